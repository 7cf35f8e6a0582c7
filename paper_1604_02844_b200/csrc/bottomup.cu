// Bottom-up levels (direction-optimising BFS; opt-in,
// not the paper's algorithm and not the headline path).
//
// A bottom-up step from frontier F_L (bitmap `front`, written by k_compact or
// rebuilt from the queues) visits every vertex v that is still unvisited and
// takes the first neighbour u of v with u in F_L as its parent (any such u is
// one level up, so the tree check of traversal.py:145-147 / validate.py holds);
// v then belongs to F_{L+1}. The visited set, the levels (written by k_compact
// from visited & ~prev as for a top-down level) and the K6 layer record
// (input = |F_L|, edges = sum of degrees of F_L, discovered = |F_{L+1}|,
// traversal.py:100) are exactly those of a top-down level: only the work
// differs (rows of unvisited vertices, cut short at the first hit, instead of
// every row of the frontier). Rows are in descending-degree order, so the
// hubs, which are in the frontier early, come first in every row.
#include "bfs_engine.cuh"

namespace lbfs {

// one warp per visited word: lane = bit = vertex; a lane scans its row four
// entries at a time (loads of the four entries, then of their frontier
// words, in flight together) until the first frontier neighbour. The warp is
// the only writer of its visited word in this step.
__global__ void __launch_bounds__(256) k_bottom_up(const BottomUpArgs b) {
  constexpr unsigned kAll = 0xFFFFFFFFu;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < b.nwords; w += nwarps) {
    const uint32_t vis = __ldcg(b.visited + w);
    const int64_t v = w * 32 + lane;
    const bool cand = !((vis >> lane) & 1u) && v < b.t_nz;
    if (!__any_sync(kAll, cand)) continue;
    int64_t p = cand ? __ldg(b.row_ptr + v) : 0, e = cand ? __ldg(b.row_ptr + v + 1) : 0;
    int32_t par = -1;
    while (p < e && par < 0) {
      int32_t u[4];
      uint32_t f[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = p + q < e ? __ldg(b.col_idx + p + q) : -1;
#pragma unroll
      for (int q = 0; q < 4; ++q) f[q] = u[q] >= 0 ? __ldg(b.front + (u[q] >> 5)) : 0u;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (par < 0 && u[q] >= 0 && ((f[q] >> (u[q] & 31)) & 1u)) par = u[q];
      p += 4;
    }
    const bool found = par >= 0;
    const uint32_t nb = __ballot_sync(kAll, found);
    if (found) b.pred_int[v] = __ldg(b.new2old + par);
    if (lane == 0 && nb) b.visited[w] = vis | nb;
  }
}

// Frontier bitmap of a queue-mode frontier (a bottom-up step right after a
// queue level): the small and warp queues hold internal ids, hub items the
// original id of their row.
__global__ void k_front_from_queues(uint32_t* __restrict__ front, const int32_t* __restrict__ qs, int64_t ns,
                                    const int32_t* __restrict__ qw, int64_t nw, const CtaItem* __restrict__ qc,
                                    int64_t nc, const int32_t* __restrict__ old2new) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns + nw + nc; i += stride) {
    int32_t v;
    if (i < ns) v = __ldcg(qs + i);
    else if (i < ns + nw) v = __ldcg(qw + (i - ns));
    else v = __ldg(old2new + __ldcg(&qc[i - ns - nw].u));
    atomicOr(front + (v >> 5), 1u << (v & 31));
  }
}

}  // namespace lbfs
