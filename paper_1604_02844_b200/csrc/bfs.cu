// Top-down BFS on sm_100a: the hot path of the reference's run_bfs
// (traversal.py:413-422 -> bfs_serial / bfs_parallel_naive / _bitmap_bfs,
// traversal.py:80-389).
//
//   K4 k_init / k_seed   PredecessorArray fill + Bitmap clear + root seed
//                        (traversal.py:42-46, 135-139, 343-347)
//   K1 k_expand<Mode>    frontier expansion over CSR, degree-binned in one
//                        launch: CTA bin (hub slices staged in shared memory
//                        by cp.async.bulk + mbarrier, double-buffered), warp
//                        bin (warp per vertex, 128-bit col_idx loads with the
//                        Listing-1 peel/body/remainder split), small bin
//                        (warp per 32 vertices over their concatenated rows).
//                        Replaces _frontier_neighbors + the 16-lane Listing-1
//                        gather (traversal.py:107-119, 297-332).
//   K2 claim             visited test-and-set: L1-cached load, then 32-bit
//                        atomicOr; the unique winner writes pred (and level in
//                        queue mode). Replaces the unsynchronised OR + negative
//                        marks + restoration pass (traversal.py:175-279).
//   K3 next frontier     two forms, chosen per level by the driver:
//                        - queue mode (small levels): warp-aggregated
//                          ballot/popc append straight from the winners;
//                        - bitmap mode (large levels): k_compact turns the
//                          newly set visited bits into the three bins with
//                          block-aggregated appends (one atomic per bin per
//                          block) and writes their levels.
//                        Replaces the np.unique merge / nonzero-word scans
//                        (traversal.py:157-158, 168-172, 366-384).
//   K5 BfsEngine::run    level driver (the while loops traversal.py:90,152,366)
//   K6 Counters          LayerStats(input, edges, discovered) per level
//                        (traversal.py:66-70, 100, 159, 383)
#include <algorithm>
#include <cstring>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "bfs_engine.cuh"

namespace lbfs {

constexpr unsigned kFull = 0xFFFFFFFFu;
enum Mode : int { kBitmapOut = 0, kQueueOut = 1 };

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int4 ld_stream4(const int32_t* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ int64_t ld_na64(const int64_t* p) {
  int64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// ---------------------------------------------------------------- TMA bulk copy
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- K2 + K3
struct Acc {  // per-thread K6 accumulators (queue mode), reduced per warp at exit
  unsigned long long disc = 0;
  unsigned long long edges = 0;
};

__device__ __forceinline__ bool bit_clear(uint32_t word, int32_t v) { return ((word >> (v & 31)) & 1u) == 0; }

// Bitmap mode: a lane whose probe saw a clear bit tries the atomic; the
// winner writes the predecessor. Levels are written by k_compact.
__device__ __forceinline__ void settle_bitmap(const LevelArgs& a, bool cand, int32_t v, int32_t u_orig) {
  if (cand) {
    const uint32_t bit = 1u << (v & 31);
    if ((atomicOr(a.visited + (v >> 5), bit) & bit) == 0) a.pred[__ldg(a.new2old + v)] = u_orig;
  }
}

__device__ __forceinline__ void warp_append(bool take, int32_t val, unsigned long long* tail, int32_t* q,
                                            int lane) {
  const unsigned m = __ballot_sync(kFull, take);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(tail, (unsigned long long)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (take) q[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// Queue mode (warp-collective): winners write level + pred, then append to
// the next level's bin with one atomic per warp per bin.
__device__ __forceinline__ void settle_queue(const LevelArgs& a, bool cand, int32_t v, int32_t u_orig, int lane,
                                             Acc& acc) {
  bool win = false;
  if (cand) {
    const uint32_t bit = 1u << (v & 31);
    win = (atomicOr(a.visited + (v >> 5), bit) & bit) == 0;
  }
  if (!__any_sync(kFull, win)) return;
  int32_t deg = 0;
  int32_t vo = 0;
  if (win) {
    atomicOr(a.prev + (v >> 5), 1u << (v & 31));  // keep bitmap-mode compaction exact
    vo = __ldg(a.new2old + v);
    a.level[vo] = a.next_level;
    a.pred[vo] = u_orig;
    deg = (int32_t)(a.row_ptr[v + 1] - a.row_ptr[v]);
    acc.disc += 1;
    acc.edges += (unsigned long long)deg;
  }
  warp_append(win && v >= a.t_warp && v < a.t_nz, v, &a.next_cnt->bin[kBinSmall], a.next_small, lane);
  warp_append(win && v >= a.t_cta && v < a.t_warp, v, &a.next_cnt->bin[kBinWarp], a.next_warp, lane);
  const int items = (win && v < a.t_cta) ? (deg + kChunk - 1) / kChunk : 0;
  if (__any_sync(kFull, items > 0)) {
    int incl = items;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    unsigned long long base = 0;
    if (lane == 31) base = atomicAdd(&a.next_cnt->bin[kBinCta], (unsigned long long)total);
    base = __shfl_sync(kFull, base, 31);
    const int off = incl - items;
    for (int k = 0; k < items; ++k)
      a.next_cta[base + off + k] = CtaItem{v, k * kChunk, min(kChunk, deg - k * kChunk), vo};
  }
}

template <int M>
__device__ __forceinline__ void settle(const LevelArgs& a, bool cand, int32_t v, int32_t u_orig, int lane, Acc& acc) {
  if constexpr (M == kBitmapOut)
    settle_bitmap(a, cand, v, u_orig);
  else
    settle_queue(a, cand, v, u_orig, lane, acc);
}

// Probe a batch of K neighbours: all K bitmap loads are issued before any
// atomic so each lane keeps K requests in flight.
template <int M, int K>
__device__ __forceinline__ void probe_batch(const LevelArgs& a, const int32_t (&nb)[K], const bool (&ok)[K],
                                            const int32_t (&par)[K], int lane, Acc& acc) {
  uint32_t w[K];
#pragma unroll
  for (int k = 0; k < K; ++k) w[k] = ok[k] ? __ldca(a.visited + (nb[k] >> 5)) : ~0u;
#pragma unroll
  for (int k = 0; k < K; ++k) settle<M>(a, ok[k] && bit_clear(w[k], nb[k]), nb[k], par[k], lane, acc);
}

template <int M>
__device__ __forceinline__ void flush_acc(const LevelArgs& a, Acc& acc) {
  if constexpr (M == kQueueOut) {
    unsigned long long d = acc.disc, e = acc.edges;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      d += __shfl_xor_sync(kFull, d, o);
      e += __shfl_xor_sync(kFull, e, o);
    }
    if ((threadIdx.x & 31) == 0 && d) {
      atomicAdd(&a.next_cnt->discovered, d);
      atomicAdd(&a.next_cnt->edges, e);
    }
  }
}

// ---------------------------------------------------------------- K1
// Warp-cooperative expansion of row [st, en) of parent u: 128-bit aligned
// body loads, scalar peel/remainder (Listing-1 split, lane.py:100-108).
template <int M>
__device__ __forceinline__ void expand_row_warp(const LevelArgs& a, int32_t u_orig, int64_t st, int64_t en,
                                                int lane, Acc& acc) {
  const int64_t al = std::min<int64_t>((st + 3) & ~int64_t(3), en);
  const int64_t bl = std::max<int64_t>(al, en & ~int64_t(3));
  {  // peel [st, al) on lanes 0..2 and remainder [bl, en) on lanes 3..5, one batch
    int64_t j = -1;
    if (lane < 3 && st + lane < al) j = st + lane;
    if (lane >= 3 && lane < 6 && bl + (lane - 3) < en) j = bl + (lane - 3);
    int32_t nb[1] = {j >= 0 ? ld_stream(a.col_idx + j) : 0};
    bool ok[1] = {j >= 0};
    int32_t par[1] = {u_orig};
    probe_batch<M, 1>(a, nb, ok, par, lane, acc);
  }
  for (int64_t j0 = al; j0 < bl; j0 += 256) {  // 2 x int4 per lane per step
    const int64_t j1 = j0 + lane * 4, j2 = j0 + 128 + lane * 4;
    const bool b1 = j1 < bl, b2 = j2 < bl;
    int4 x = b1 ? ld_stream4(a.col_idx + j1) : make_int4(0, 0, 0, 0);
    int4 y = b2 ? ld_stream4(a.col_idx + j2) : make_int4(0, 0, 0, 0);
    int32_t nb[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
    bool ok[8] = {b1, b1, b1, b1, b2, b2, b2, b2};
    int32_t par[8] = {u_orig, u_orig, u_orig, u_orig, u_orig, u_orig, u_orig, u_orig};
    probe_batch<M, 8>(a, nb, ok, par, lane, acc);
  }
}

struct CtaMeta {
  int32_t shift;  // first valid element within the staged buffer
  int32_t len;
  int32_t u_orig;
  int32_t nvec;   // int4 slots staged
};

template <int M>
__global__ void __launch_bounds__(kExpandThreads, 4) k_expand(LevelArgs a, Frontier f) {
  __shared__ alignas(128) int32_t s_buf[2][kChunk + 8];
  __shared__ alignas(8) uint64_t s_bar[2];
  __shared__ CtaMeta s_meta[2];
  __shared__ int32_t s_off[kExpandThreads / 32][33];
  __shared__ int64_t s_start[kExpandThreads / 32][32];
  __shared__ int32_t s_par[kExpandThreads / 32][32];
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  Acc acc;

  // ---- phase 1: CTA bin, TMA-staged kChunk-edge hub slices ---------------
  if (f.n_cta > (int64_t)blockIdx.x) {
    if (tid == 0) {
      mbar_init(&s_bar[0], 1);
      mbar_init(&s_bar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t it, int b) {  // thread 0
      const CtaItem c = f.cta[it];
      const int64_t st = a.row_ptr[c.v] + c.off;
      const int64_t a0 = st & ~int64_t(3);
      const int64_t a1 = (st + c.len + 3) & ~int64_t(3);
      const uint32_t bytes = (uint32_t)((a1 - a0) * 4);
      s_meta[b] = CtaMeta{(int32_t)(st - a0), c.len, c.v_orig, (int32_t)((a1 - a0) / 4)};
      mbar_expect_tx(&s_bar[b], bytes);
      bulk_g2s(&s_buf[b][0], a.col_idx + a0, bytes, &s_bar[b]);
    };
    if (tid == 0) issue(blockIdx.x, 0);
    __syncthreads();
    uint32_t ph[2] = {0u, 0u};
    int b = 0;
    for (int64_t it = blockIdx.x; it < f.n_cta; it += gridDim.x) {
      if (tid == 0 && it + gridDim.x < f.n_cta) issue(it + gridDim.x, b ^ 1);
      mbar_wait(&s_bar[b], ph[b]);
      ph[b] ^= 1u;
      const CtaMeta m = s_meta[b];
      const int4* v4 = reinterpret_cast<const int4*>(&s_buf[b][0]);
      for (int base = 0; base < m.nvec; base += 2 * kExpandThreads) {
        const int s1 = base + tid, s2 = base + kExpandThreads + tid;
        const int4 x = s1 < m.nvec ? v4[s1] : make_int4(0, 0, 0, 0);
        const int4 y = s2 < m.nvec ? v4[s2] : make_int4(0, 0, 0, 0);
        int32_t nb[8] = {x.x, x.y, x.z, x.w, y.x, y.y, y.z, y.w};
        bool ok[8];
        int32_t par[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int e = (k < 4 ? s1 * 4 + k : s2 * 4 + (k - 4)) - m.shift;
          ok[k] = (k < 4 ? s1 < m.nvec : s2 < m.nvec) && e >= 0 && e < m.len;
          par[k] = m.u_orig;
        }
        probe_batch<M, 8>(a, nb, ok, par, lane, acc);
      }
      __syncthreads();  // buffer b is free again
      b ^= 1;
    }
  }

  const int64_t gwarp = ((int64_t)blockIdx.x * blockDim.x + tid) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;

  // ---- phase 2: warp bin, one warp per vertex ------------------------------
  for (int64_t i = gwarp; i < f.n_warp; i += nwarps) {
    const int32_t u = f.warp[i];
    const int64_t st = a.row_ptr[u], en = a.row_ptr[u + 1];
    expand_row_warp<M>(a, __ldg(a.new2old + u), st, en, lane, acc);
  }

  // ---- phase 3: small bin, a warp walks 32 vertices' concatenated rows ----
  for (int64_t base = gwarp * 32; base < f.n_small; base += nwarps * 32) {
    const int64_t i = base + lane;
    int64_t st = 0;
    int32_t d = 0, uo = 0;
    if (i < f.n_small) {
      const int32_t u = f.small[i];
      st = a.row_ptr[u];
      d = (int32_t)(a.row_ptr[u + 1] - st);
      uo = __ldg(a.new2old + u);
    }
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    s_off[wib][lane] = incl - d;
    s_start[wib][lane] = st;
    s_par[wib][lane] = uo;
    __syncwarp();
    for (int e0 = 0; e0 < total; e0 += 128) {
      int32_t nb[4], par[4];
      bool ok[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int e = e0 + k * 32 + lane;
        ok[k] = e < total;
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1)
          if (s_off[wib][lo + step] <= e) lo += step;
        nb[k] = ok[k] ? ld_stream(a.col_idx + s_start[wib][lo] + (e - s_off[wib][lo])) : 0;
        par[k] = s_par[wib][lo];
      }
      probe_batch<M, 4>(a, nb, ok, par, lane, acc);
    }
    __syncwarp();
  }
  flush_acc<M>(a, acc);
}

// ---------------------------------------------------------------- K3 compaction
// One thread per visited word: new = visited & ~prev. Each block scans its
// per-bin counts, takes one atomic per bin, writes its entries in ascending
// internal id, writes the new vertices' levels and folds the K6 stats.
constexpr int kCompactThreads = 256;

__device__ __forceinline__ uint32_t range_mask(int64_t base_v, int64_t lo, int64_t hi) {
  // bits b with lo <= base_v + b < hi
  const int64_t a = std::max<int64_t>(lo - base_v, 0), b = std::min<int64_t>(hi - base_v, 32);
  if (a >= b) return 0u;
  const uint32_t hi_m = (b >= 32) ? kFull : ((1u << b) - 1u);
  const uint32_t lo_m = (a >= 32) ? kFull : ((1u << a) - 1u);
  return hi_m & ~lo_m;
}

__global__ void __launch_bounds__(kCompactThreads) k_compact(CompactArgs c) {
  using Scan = cub::BlockScan<unsigned long long, kCompactThreads>;
  using Reduce = cub::BlockReduce<unsigned long long, kCompactThreads>;
  __shared__ typename Scan::TempStorage s_scan;
  __shared__ typename Reduce::TempStorage s_red;
  __shared__ unsigned long long s_base[3];
  const int64_t i = (int64_t)blockIdx.x * kCompactThreads + threadIdx.x;
  uint32_t nb = 0;
  if (i < c.nwords) {
    const uint32_t w = c.visited[i], p = c.prev[i];
    nb = w & ~p;
    if (nb) c.prev[i] = w;
  }
  const int64_t v0 = i * 32;
  const uint32_t m_cta = nb & range_mask(v0, 0, c.t_cta);
  const uint32_t m_warp = nb & range_mask(v0, c.t_cta, c.t_warp);
  const uint32_t m_small = nb & range_mask(v0, c.t_warp, c.t_nz);
  unsigned long long n_items = 0;
  for (uint32_t m = m_cta; m; m &= m - 1) {
    const int64_t v = v0 + __ffs(m) - 1;
    const int64_t deg = c.row_ptr[v + 1] - c.row_ptr[v];
    n_items += (unsigned long long)((deg + kChunk - 1) / kChunk);
  }
  // pack: items [0,21) | warp [21,42) | small [42,63)
  const unsigned long long packed =
      n_items | ((unsigned long long)__popc(m_warp) << 21) | ((unsigned long long)__popc(m_small) << 42);
  unsigned long long excl, total;
  Scan(s_scan).ExclusiveSum(packed, excl, total);
  if (threadIdx.x == 0) {
    const unsigned long long t_items = total & 0x1FFFFF, t_warp = (total >> 21) & 0x1FFFFF,
                             t_small = (total >> 42) & 0x1FFFFF;
    s_base[0] = t_small ? atomicAdd(&c.next_cnt->bin[kBinSmall], t_small) : 0;
    s_base[1] = t_warp ? atomicAdd(&c.next_cnt->bin[kBinWarp], t_warp) : 0;
    s_base[2] = t_items ? atomicAdd(&c.next_cnt->bin[kBinCta], t_items) : 0;
  }
  __syncthreads();
  unsigned long long p_items = s_base[2] + (excl & 0x1FFFFF);
  unsigned long long p_warp = s_base[1] + ((excl >> 21) & 0x1FFFFF);
  unsigned long long p_small = s_base[0] + ((excl >> 42) & 0x1FFFFF);
  unsigned long long edges = 0;
  for (uint32_t m = nb; m; m &= m - 1) {
    const int b = __ffs(m) - 1;
    const int64_t v = v0 + b;
    const int32_t vo = c.new2old[v];
    c.level[vo] = c.next_level;
    const int64_t st = c.row_ptr[v];
    const int64_t deg = c.row_ptr[v + 1] - st;
    edges += (unsigned long long)deg;
    const uint32_t bit = 1u << b;
    if (m_small & bit) {
      c.next_small[p_small++] = (int32_t)v;
    } else if (m_warp & bit) {
      c.next_warp[p_warp++] = (int32_t)v;
    } else if (m_cta & bit) {
      for (int64_t k = 0; k * kChunk < deg; ++k)
        c.next_cta[p_items++] = CtaItem{(int32_t)v, (int32_t)(k * kChunk),
                                        (int32_t)std::min<int64_t>(kChunk, deg - k * kChunk), vo};
    }
  }
  const unsigned long long e_tot = Reduce(s_red).Sum(edges);
  __syncthreads();
  const unsigned long long d_tot = Reduce(s_red).Sum((unsigned long long)__popc(nb));
  if (threadIdx.x == 0) {
    if (e_tot) atomicAdd(&c.next_cnt->edges, e_tot);
    if (d_tot) atomicAdd(&c.next_cnt->discovered, d_tot);
  }
}

// ---------------------------------------------------------------- K4 init
__global__ void k_init(int32_t* __restrict__ pred, int64_t npad, int32_t* __restrict__ level, int64_t n,
                       uint32_t* __restrict__ visited, uint32_t* __restrict__ prev, int64_t nwords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t; i < npad; i += stride) pred[i] = kSentinel;
  for (int64_t i = t; i < n; i += stride) level[i] = -1;
  for (int64_t i = t; i < nwords; i += stride) visited[i] = prev[i] = 0;
}

__global__ void k_init_vec(int4* __restrict__ pred4, int64_t npad4, int4* __restrict__ level4, int64_t n4,
                           int32_t* __restrict__ level, int64_t n, uint4* __restrict__ vis4,
                           uint4* __restrict__ prev4, int64_t nwords4) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int4 s4 = make_int4(kSentinel, kSentinel, kSentinel, kSentinel);
  const int4 m4 = make_int4(-1, -1, -1, -1);
  for (int64_t i = t; i < npad4; i += stride) pred4[i] = s4;
  for (int64_t i = t; i < n4; i += stride) level4[i] = m4;
  for (int64_t i = 4 * n4 + t; i < n; i += stride) level[i] = -1;
  for (int64_t i = t; i < nwords4; i += stride) vis4[i] = prev4[i] = make_uint4(0, 0, 0, 0);
}

__global__ void k_seed(LevelArgs a, uint32_t* prev, const int32_t* old2new, int32_t root_orig, Counters* cnt0) {
  const int32_t r = old2new[root_orig];
  const int64_t st = a.row_ptr[r];
  const int32_t deg = (int32_t)(a.row_ptr[r + 1] - st);
  a.visited[r >> 5] |= 1u << (r & 31);
  prev[r >> 5] |= 1u << (r & 31);
  a.level[root_orig] = 0;
  a.pred[root_orig] = root_orig;
  Counters c{};
  c.discovered = 1;
  c.edges = (unsigned long long)deg;
  if (r < a.t_cta) {
    const int items = (deg + kChunk - 1) / kChunk;
    for (int k = 0; k < items; ++k) a.next_cta[k] = CtaItem{r, k * kChunk, min(kChunk, deg - k * kChunk), root_orig};
    c.bin[kBinCta] = (unsigned long long)items;
  } else if (r < a.t_warp) {
    a.next_warp[0] = r;
    c.bin[kBinWarp] = 1;
  } else if (r < a.t_nz) {
    a.next_small[0] = r;
    c.bin[kBinSmall] = 1;
  }
  *cnt0 = c;
}

// ---------------------------------------------------------------- engine
BfsEngine::BfsEngine(const Csr& csr) {
  LBFS_CUDA(cudaGetDevice(&device_));
  sm_count_ = current_sm_count();
  n_ = csr.n;
  nnz_ = csr.nnz;
  nwords_ = (n_ + 31) / 32;
  npad_ = pad32(n_);
  LBFS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  build_layout(csr);
  visited_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
  prev_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
  // Bins, double-buffered: a vertex enters a bin once per BFS, so n entries
  // bound the small/warp bins; CTA items <= nnz/kChunk + #(deg >= kCtaMin).
  cap_cta_ = nnz_ / kChunk + t_cta_ + 2;
  for (int b = 0; b < 2; ++b) {
    q_small_[b] = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_, 1));
    q_warp_[b] = dev_alloc<int32_t>((size_t)std::max<int64_t>(t_warp_, 1));
    q_cta_[b] = dev_alloc<CtaItem>((size_t)cap_cta_);
  }
  cnt_ = dev_alloc<Counters>(kCounterRing);
  LBFS_CUDA(cudaMallocHost(&h_cnt_, sizeof(Counters) * kCounterRing));
  for (auto& e : ev_) LBFS_CUDA(cudaEventCreate(&e));
  int occ = 0;
  LBFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_expand<kBitmapOut>, kExpandThreads, 0));
  expand_grid_ = sm_count_ * std::max(occ, 1);
}

BfsEngine::~BfsEngine() {
  cudaStreamSynchronize(stream_);
  dev_free(visited_);
  dev_free(prev_);
  for (int b = 0; b < 2; ++b) {
    dev_free(q_small_[b]);
    dev_free(q_warp_[b]);
    dev_free(q_cta_[b]);
  }
  dev_free(cnt_);
  if (h_cnt_) cudaFreeHost(h_cnt_);
  dev_free(own_pred_);
  dev_free(own_level_);
  for (auto& e : ev_) cudaEventDestroy(e);
  dev_free(row_ptr_);
  dev_free(col_idx_);
  dev_free(new2old_);
  dev_free(old2new_);
  cudaStreamDestroy(stream_);
}

void BfsEngine::ensure_own_outputs() {
  if (!own_pred_) own_pred_ = dev_alloc<int32_t>((size_t)npad_);
  if (!own_level_) own_level_ = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_, 1));
}

static unsigned clamp_grid(int64_t blocks, int64_t cap) {
  return (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
}

void BfsEngine::run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t) {
  if (root < 0 || root >= n_) throw_inval("root out of range");
  const int64_t launches0 = g_launches.load();
  cudaStream_t st = stream_;
  LBFS_CUDA(cudaEventRecord(ev_[0], st));
  {  // K4
    const bool aligned = ((uintptr_t)d_pred % 16 == 0) && ((uintptr_t)d_level % 16 == 0);
    const unsigned grid = clamp_grid((npad_ / 4 + 255) / 256, (int64_t)sm_count_ * 8);
    if (aligned && nwords_ % 4 == 0) {
      LBFS_LAUNCH(k_init_vec, grid, 256, 0, st, (int4*)d_pred, npad_ / 4, (int4*)d_level, n_ / 4, d_level, n_,
                  (uint4*)visited_, (uint4*)prev_, nwords_ / 4);
    } else {
      LBFS_LAUNCH(k_init, grid, 256, 0, st, d_pred, npad_, d_level, n_, visited_, prev_, nwords_);
    }
  }
  LevelArgs a{};
  a.row_ptr = row_ptr_;
  a.col_idx = col_idx_;
  a.new2old = new2old_;
  a.visited = visited_;
  a.prev = prev_;
  a.pred = d_pred;
  a.level = d_level;
  a.t_cta = t_cta_;
  a.t_warp = t_warp_;
  a.t_nz = t_nz_;
  int cur = 0;
  a.next_small = q_small_[cur];
  a.next_warp = q_warp_[cur];
  a.next_cta = q_cta_[cur];
  LBFS_LAUNCH(k_seed, 1, 1, 0, st, a, prev_, old2new_, (int32_t)root, &cnt_[0]);
  LBFS_CUDA(cudaMemcpyAsync(&h_cnt_[0], &cnt_[0], sizeof(Counters), cudaMemcpyDeviceToHost, st));
  LBFS_CUDA(cudaEventRecord(ev_[1], st));
  LBFS_CUDA(cudaStreamSynchronize(st));

  layers_.clear();
  double expand_ms = 0.0;
  const unsigned long long bitmap_min_edges = (unsigned long long)std::max<int64_t>(1 << 16, n_ / 64);
  int64_t L = 0;
  for (;;) {
    const Counters c = h_cnt_[L % kCounterRing];
    const int slot = (int)((L + 1) % kCounterRing);
    LBFS_CUDA(cudaMemsetAsync(&cnt_[slot], 0, sizeof(Counters), st));
    a.next_level = (int32_t)(L + 1);
    a.next_cnt = &cnt_[slot];
    a.next_small = q_small_[cur ^ 1];
    a.next_warp = q_warp_[cur ^ 1];
    a.next_cta = q_cta_[cur ^ 1];
    Frontier f{q_small_[cur], q_warp_[cur], q_cta_[cur], (int64_t)c.bin[kBinSmall], (int64_t)c.bin[kBinWarp],
               (int64_t)c.bin[kBinCta]};
    const bool bitmap = c.edges >= bitmap_min_edges;
    const int64_t need = std::max({f.n_cta, (f.n_warp + 7) / 8, (f.n_small + 255) / 256, (int64_t)1});
    const unsigned grid = clamp_grid(need, expand_grid_);
    LBFS_CUDA(cudaEventRecord(ev_[2], st));
    if (f.n_cta + f.n_warp + f.n_small > 0) {
      if (bitmap) {
        LBFS_LAUNCH(k_expand<kBitmapOut>, grid, kExpandThreads, 0, st, a, f);
      } else {
        LBFS_LAUNCH(k_expand<kQueueOut>, grid, kExpandThreads, 0, st, a, f);
      }
    }
    LBFS_CUDA(cudaEventRecord(ev_[3], st));
    if (bitmap) {
      CompactArgs ca{row_ptr_, new2old_, visited_, prev_, nwords_, d_level, (int32_t)(L + 1), t_cta_, t_warp_, t_nz_,
                     &cnt_[slot], q_small_[cur ^ 1], q_warp_[cur ^ 1], q_cta_[cur ^ 1]};
      LBFS_LAUNCH(k_compact, (unsigned)((nwords_ + kCompactThreads - 1) / kCompactThreads), kCompactThreads, 0, st,
                  ca);
    }
    LBFS_CUDA(cudaMemcpyAsync(&h_cnt_[slot], &cnt_[slot], sizeof(Counters), cudaMemcpyDeviceToHost, st));
    LBFS_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
    expand_ms += ms;
    const Counters nx = h_cnt_[slot];
    layers_.push_back(lbfs_layer{(int64_t)c.discovered, (int64_t)c.edges, (int64_t)nx.discovered});
    cur ^= 1;
    ++L;
    if (nx.discovered == 0) break;
  }
  LBFS_CUDA(cudaEventRecord(ev_[4], st));
  LBFS_CUDA(cudaEventSynchronize(ev_[4]));
  if (t) {
    float total = 0.f, init = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&total, ev_[0], ev_[4]));
    LBFS_CUDA(cudaEventElapsedTime(&init, ev_[0], ev_[1]));
    t->bfs_ms = total;
    t->init_ms = init;
    t->expand_ms = expand_ms;
    t->d2h_ms = 0.0;
    t->levels = (int64_t)layers_.size();
    t->kernel_launches = g_launches.load() - launches0;
    int64_t e = 0, r = 0;
    for (auto& l : layers_) {
      e += l.edges;
      r += l.input;
    }
    t->edges = e;
    t->reached = r;
  }
}

}  // namespace lbfs
