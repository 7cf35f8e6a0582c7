// Heavy levels as one streaming pass over the whole CSR (K1 + K2 for the
// levels that carry most of the graph's edges: the reference's
// _frontier_neighbors + Listing-1 gather + bitmap test-and-set,
// traversal.py:107-119, 175-193, 297-332).
//
// At a heavy level most rows are in the frontier, so instead of per-row work
// lists the rows of degree >= 1 — one contiguous col_idx range [0, e_nz) in
// the degree-ordered layout — are cut into 128-element windows and streamed
// whole:
//
//   k_window_masks   one thread per big-row window: the rows it touches (the
//                    side entry: row of its first element + <= 4 row starts)
//                    and their frontier bits -> its 128-bit valid mask; the
//                    small-row windows come from k_sweep_plan_small (closed-
//                    form rows per degree class, sweep.cu)
//   k_stream_heavy   every warp of the GPU takes an equal contiguous range of
//                    windows; per window a lane reads its 4-bit slice of the
//                    mask and, when nonzero, its 16 bytes of col_idx. The
//                    masks of the next-but-one group and the data of the next
//                    group are in flight while a group is processed. Valid
//                    targets are OR'ed blindly (heavy semantics: no probe, no
//                    parent): hot ids into the CTA's shared copy of the hot
//                    prefix (later folded into visited by k_merge_hot), cold
//                    ids into visited in L2 (fire and forget); consecutive
//                    targets of a lane in one bitmap word take one OR.
//
// No producer warps, no shared-memory staging of the stream: shared memory
// holds only the hot prefix (longer than the TMA-ring sweep's), and the
// in-flight bytes per SM come from 32 warps x 2 groups x D windows.
#include "bfs_engine.cuh"

namespace lbfs {

namespace {

constexpr int kWin = kSweepWindow;  // elements per window
constexpr unsigned kAll = 0xFFFFFFFFu;

__device__ __forceinline__ int4 ld_nc4(const int32_t* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void red_or_g(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_s(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// bits [lo, hi) of word k of a 128-bit mask
__device__ __forceinline__ uint32_t range_word(int lo, int hi, int k) {
  const int a = max(lo - 32 * k, 0), b = min(hi - 32 * k, 32);
  if (a >= b) return 0u;
  const uint32_t hm = b >= 32 ? kAll : (1u << b) - 1u;
  return hm & ~((1u << a) - 1u);
}

}  // namespace

// Valid masks of the big-row windows [0, nwin): element o of window w is
// valid when its row is in the frontier and w * 128 + o < e_big. The window
// holding e_big also takes the small-row part of its mask (svmask[0] when it
// is window w_small0).
__global__ void k_window_masks(const uint2* __restrict__ side, int64_t nwin, int64_t e_big,
                               const uint32_t* __restrict__ front, const uint4* __restrict__ svmask, int64_t w_small0,
                               uint4* __restrict__ wmask) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const uint2 sd = __ldg(side + w);
    const uint32_t r0 = sd.x;
    const uint64_t f64 = ((uint64_t)__ldg(front + (r0 >> 5) + 1) << 32) | __ldg(front + (r0 >> 5));
    const uint32_t fb = (uint32_t)(f64 >> (r0 & 31));  // frontier bits of rows r0 .. r0 + 4
    const int lim = (int)min((int64_t)kWin, e_big - w * kWin);
    uint32_t m[4] = {0u, 0u, 0u, 0u};
    int lo = 0;
#pragma unroll
    for (int r = 0; r < 5; ++r) {
      const int st = r < 4 ? (int)((sd.y >> (8 * r)) & 0xFFu) : 0xFF;  // start of row r0 + r + 1
      const int hi = min(min(st, kWin), lim);
      if ((fb >> r) & 1u) {
#pragma unroll
        for (int k = 0; k < 4; ++k) m[k] |= range_word(lo, hi, k);
      }
      lo = max(lo, min(st, kWin));
    }
    if (w == w_small0 && svmask) {
      const uint4 s = __ldg(svmask);
      m[0] |= s.x, m[1] |= s.y, m[2] |= s.z, m[3] |= s.w;
    }
    wmask[w] = make_uint4(m[0], m[1], m[2], m[3]);
  }
}

// dynamic shared memory: the hot prefix (hot_words words, zeroed here)
template <int D>
__global__ void __launch_bounds__(kStreamThreads, 1) k_stream_heavy(const __grid_constant__ StreamArgs s) {
  extern __shared__ __align__(16) uint32_t s_hot[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int hw4 = s.hot_words >> 2;
  uint4* h4 = reinterpret_cast<uint4*>(s_hot);
  for (int i = tid; i < hw4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint32_t hoff = (uint32_t)__cvta_generic_to_shared(s_hot);
  // this warp's windows: an equal contiguous share (warps interleave the SMs)
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t gw = (int64_t)(tid >> 5) * gridDim.x + blockIdx.x;
  const int64_t w_beg = s.nwin * gw / nw, w_end = s.nwin * (gw + 1) / nw;
  const uint32_t* wm32 = reinterpret_cast<const uint32_t*>(s.wmask);
  const uint32_t* sv32 = reinterpret_cast<const uint32_t*>(s.svmask);
  const int sh = 4 * (lane & 7), mw = lane >> 3;
  // this lane's 4 mask bits of window w
  auto nib = [&](int64_t w) -> uint32_t {
    if (w >= w_end) return 0u;
    const uint32_t word = w < s.nwin_big ? __ldg(wm32 + 4 * w + mw) : __ldg(sv32 + 4 * (w - s.w_small0) + mw);
    return (word >> sh) & 0xFu;
  };
  auto data = [&](int64_t w, uint32_t nb) -> int4 {
    return nb ? ld_nc4(s.col_idx + w * kWin + lane * 4) : make_int4(0, 0, 0, 0);
  };
  uint32_t ma[D], mb[D];
  int4 xa[D];
#pragma unroll
  for (int d = 0; d < D; ++d) ma[d] = nib(w_beg + d);
#pragma unroll
  for (int d = 0; d < D; ++d) xa[d] = data(w_beg + d, ma[d]);
#pragma unroll
  for (int d = 0; d < D; ++d) mb[d] = nib(w_beg + D + d);
  for (int64_t w = w_beg; w < w_end; w += D) {
    int4 xb[D];
    uint32_t mc[D];
#pragma unroll
    for (int d = 0; d < D; ++d) xb[d] = data(w + D + d, mb[d]);
#pragma unroll
    for (int d = 0; d < D; ++d) mc[d] = nib(w + 2 * D + d);
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const uint32_t m = ma[d];
      if (!m) continue;
      const int32_t e[4] = {xa[d].x, xa[d].y, xa[d].z, xa[d].w};
      int32_t run_w = -1;
      uint32_t run_b = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!((m >> q) & 1u)) continue;
        const int32_t wi = e[q] >> 5;
        const uint32_t bit = 1u << (e[q] & 31);
        if (wi == run_w) {
          run_b |= bit;
          continue;
        }
        if (run_b) {
          if (run_w < s.hot_words) red_or_s(hoff + 4u * (uint32_t)run_w, run_b);
          else red_or_g(s.visited + run_w, run_b);
        }
        run_w = wi;
        run_b = bit;
      }
      if (run_b) {
        if (run_w < s.hot_words) red_or_s(hoff + 4u * (uint32_t)run_w, run_b);
        else red_or_g(s.visited + run_w, run_b);
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      ma[d] = mb[d];
      mb[d] = mc[d];
      xa[d] = xb[d];
    }
  }
  __syncthreads();
  uint4* row = reinterpret_cast<uint4*>(s.stage) + (size_t)blockIdx.x * (s.stage_words >> 2);
  for (int i = tid; i < hw4; i += blockDim.x) __stcg(row + i, h4[i]);
}

template __global__ void k_stream_heavy<kStreamDepth>(const __grid_constant__ StreamArgs s);

}  // namespace lbfs
