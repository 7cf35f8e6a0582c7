// Heavy-level sweep of the big-row region (K1 + K2 for the levels that carry
// most of the graph's edges; the reference's _frontier_neighbors + Listing-1
// gather + the bitmap test-and-set, traversal.py:107-119, 175-193, 297-332).
//
// Rows of degree >= 32 (internal ids [0, t_warp): hubs and warp-bin rows)
// occupy one contiguous col_idx range [0, e_big). At a heavy level most of
// those rows are in the frontier, so instead of per-row slice lists the
// region is streamed whole, in 128-element windows, with 128-bit loads. A
// per-window side entry (built once with the layout) names the row holding
// the window's first element and the offsets of the <= 4 rows starting
// inside it, so a lane finds the row of its elements without row_ptr: the
// frontier bits of those <= 5 consecutive rows decide whether the window is
// skipped (no load), taken whole, or masked per element.
//
// Per element (heavy semantics, see kHeavy in bfs.cu): a target in the hot
// prefix is OR'ed blindly into the CTA's shared copy (flushed to its stage
// row; k_merge_hot folds the rows into visited), a cold target blindly into
// visited in L2 with a fire-and-forget red.or. No parent is written: k_resolve
// gives every vertex of the level its first neighbour one level up.
//
// Warp-specialised pipeline per CTA (one per SM): producer warps read the
// side entries and frontier words of a 32-window chunk (two chunks ahead),
// write the window metadata and bulk-copy (TMA) the span of windows that hold
// frontier rows into a kSweepStages-deep shared ring; 16 consumer warps copy
// two windows each into registers, release the stage, then OR the targets,
// so no warp waits on L2 per element.
#include <algorithm>

#include "bfs_engine.cuh"

#ifndef LBFS_SWEEP_DBG
#define LBFS_SWEEP_DBG 0  // experiments (wrong results): 1 no hot ORs, 2 no cold ORs, 4 consumers skip the data
#endif

namespace lbfs {

namespace {

constexpr unsigned kAll = 0xFFFFFFFFu;
constexpr int kWin = kSweepWindow;  // elements per window
constexpr int kSweepDbg = LBFS_SWEEP_DBG;
#ifndef LBFS_SWEEP_HOTCHK
#define LBFS_SWEEP_HOTCHK 0
#endif

__device__ __forceinline__ int4 ld_stream4(const int32_t* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void red_or_g(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Window info for lanes 0..3 (window 4g + lane): 5 frontier bits of the rows
// first .. first+4 masked to the rows present, and a code (0 skip, 1 whole,
// 2 masked) in bits 8..9.
__device__ __forceinline__ uint32_t window_info(uint2 sd, uint2 fw, bool valid) {
  if (!valid) return 0u;
  int ns = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) ns += ((sd.y >> (8 * k)) & 0xFFu) != 0xFFu;
  const uint32_t sh = sd.x & 31u;
  const uint64_t f64 = ((uint64_t)fw.y << 32) | fw.x;
  const uint32_t mask = (2u << ns) - 1u;
  const uint32_t fb = (uint32_t)(f64 >> sh) & mask;
  const uint32_t code = fb == 0 ? 0u : (fb == mask ? 1u : 2u);
  return fb | (code << 8);
}

}  // namespace

__global__ void k_side_table(const int64_t* __restrict__ rp, int32_t nrows, int64_t nwin, uint2* __restrict__ side) {
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < nwin; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t P = w * kWin;
    int32_t lo = 0, hi = nrows - 1;  // last row with rp[row] <= P (rp[0] = 0)
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (rp[mid] <= P) lo = mid;
      else hi = mid - 1;
    }
    uint32_t starts = kAll;
    int k = 0;
    for (int32_t r = lo + 1; r < nrows && k < 4; ++r, ++k) {
      const int64_t s = rp[r];
      if (s >= P + kWin) break;
      starts = (starts & ~(0xFFu << (8 * k))) | ((uint32_t)(s - P) << (8 * k));
    }
    side[w] = make_uint2((uint32_t)lo, starts);
  }
}

// Small-region window descriptors (built once with the layout): for window
// w >= w0, the first small element P0 = max(128 w, e_big), its degree class
// d, row o0 = T[d+1] + (P0 - base[d]) / d and offset r0 = (P0 - base[d]) % d
// in that row; x = o0, y = d | r0 << 8 | s0 << 16 | (window crosses a class
// boundary) << 31, s0 = P0 - 128 w.
__device__ __forceinline__ int small_class(const int64_t* B, int64_t p) {
  int d = kSmallMax - 1;  // smallest d with base[d] <= p (base is non-increasing in d)
#pragma unroll
  for (int step = 16; step; step >>= 1)
    if (d - step >= 1 && B[d - step] <= p) d -= step;
  return d;
}
__global__ void k_small_desc(const ClassTable* __restrict__ classes, int64_t e_big, int64_t e_end, int64_t w0,
                             int64_t nw, uint2* __restrict__ desc) {
  __shared__ int32_t T[kSmallMax + 2];
  __shared__ int64_t B[kSmallMax + 1];
  if (threadIdx.x < kSmallMax + 2) T[threadIdx.x] = classes->T[threadIdx.x];
  if (threadIdx.x < kSmallMax + 1) B[threadIdx.x] = classes->base[threadIdx.x];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t P = (w0 + i) * kWin, P0 = P > e_big ? P : e_big;
    const int d = small_class(B, P0);
    const int64_t rel = P0 - B[d];
    const int64_t class_end = B[d] + (int64_t)(T[d] - T[d + 1]) * d;
    const uint32_t cross = (P + kWin > class_end && class_end < e_end) ? 1u : 0u;
    desc[i] = make_uint2((uint32_t)(T[d + 1] + rel / d),
                         (uint32_t)d | (uint32_t)(rel % d) << 8 | (uint32_t)(P0 - P) << 16 | cross << 31);
  }
}

// Per heavy level: valid-element masks of the small-region windows [w0,
// w0 + nw), one warp per window (a lane's 4 elements: rows in closed form
// from the window descriptor, their frontier bits through L1).
__global__ void k_sweep_plan_small(const ClassTable* __restrict__ classes, const uint2* __restrict__ desc,
                                   const uint32_t* __restrict__ front, int64_t e_end, int64_t w0, int64_t nw,
                                   uint4* __restrict__ svmask) {
  __shared__ int32_t T[kSmallMax + 2];
  __shared__ int64_t B[kSmallMax + 1];
  __shared__ uint32_t magic[kSmallMax + 1];
  if (threadIdx.x < kSmallMax + 2) T[threadIdx.x] = classes->T[threadIdx.x];
  if (threadIdx.x < kSmallMax + 1) {
    B[threadIdx.x] = classes->base[threadIdx.x];
    magic[threadIdx.x] = threadIdx.x ? (uint32_t)(0xFFFFFFFFull / threadIdx.x + 1ull) : 0u;  // x / d = umulhi(x, magic)
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // kPW windows per warp step, their loads batched (the kernel is latency-bound)
  constexpr int kPW = 8;
  for (int64_t i0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) * kPW; i0 < nw; i0 += nwarps * kPW) {
    uint2 dc[kPW];
#pragma unroll
    for (int k = 0; k < kPW; ++k) dc[k] = i0 + k < nw ? __ldg(desc + i0 + k) : make_uint2(0u, 0u);
    int32_t own[kPW][4];
    uint32_t ok = 0;
#pragma unroll
    for (int k = 0; k < kPW; ++k) {
      const int d = (int)(dc[k].y & 0xFFu), r0 = (int)((dc[k].y >> 8) & 0xFFu), s0 = (int)((dc[k].y >> 16) & 0xFFu);
      const bool cross = dc[k].y >> 31;
      const int64_t P = (w0 + i0 + k) * kWin;
      const int lim = i0 + k < nw ? (int)min((int64_t)kWin, e_end - P) : 0;  // valid offsets [s0, lim)
      // row and column of this lane's first element, then step through the other three
      const int x0 = r0 + 4 * lane - s0;
      const uint32_t q0 = d == 1 ? (uint32_t)max(x0, 0) : __umulhi((uint32_t)max(x0, 0), magic[d]);
      int32_t row = (int32_t)dc[k].x + (int32_t)q0;
      int col = max(x0, 0) - (int)q0 * d;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int off = 4 * lane + q;
        own[k][q] = row;
        if (cross && off >= s0 && off < lim) {  // (rare) the window crosses a class boundary
          const int64_t p = P + off;
          const int dd = small_class(B, p);
          own[k][q] = T[dd + 1] + (int32_t)((p - B[dd]) / dd);
        }
        ok |= (uint32_t)(off >= s0 && off < lim) << (4 * k + q);
        if (off >= s0 && ++col == d) {
          col = 0;
          ++row;
        }
      }
    }
    uint32_t fw[kPW][4];
#pragma unroll
    for (int k = 0; k < kPW; ++k)
#pragma unroll
      for (int q = 0; q < 4; ++q) fw[k][q] = ((ok >> (4 * k + q)) & 1u) ? __ldg(front + (own[k][q] >> 5)) : 0u;
#pragma unroll
    for (int k = 0; k < kPW; ++k) {
      uint32_t nib = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) nib |= ((fw[k][q] >> (own[k][q] & 31)) & 1u) << q;
      uint32_t wk[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) wk[j] = __reduce_or_sync(kAll, (lane >> 3) == j ? nib << (4 * (lane & 7)) : 0u);
      if (lane == 0 && i0 + k < nw) svmask[i0 + k] = make_uint4(wk[0], wk[1], wk[2], wk[3]);
    }
  }
}

namespace {

// CTA layout: kSweepConsumers consumer warps + 1 producer warp. The CTA
// walks chunks blockIdx.x, blockIdx.x + gridDim.x, ... of kChunkWins
// windows; chunk i goes through ring stage i % kStages.
constexpr int kChunkWins = kSweepChunkWins;          // windows per chunk (16 KB at 32)
constexpr int kConsumers = kSweepConsumers;          // consumer warps
constexpr int kWinPerWarp = kChunkWins / kConsumers;  // windows per consumer warp per chunk
constexpr int kEl = 4 * kWinPerWarp;                 // elements per consumer lane per chunk
constexpr int kStages = kSweepStages;

struct WinMeta {
  uint32_t vmask[4];  // valid elements of the window (rows in the frontier, below e_big): bit o of word o/32
  uint32_t info;      // window_info: frontier bits | code << 8
  uint32_t pad[3];
};

// bits [lo, hi) of word k of a 128-bit mask
__device__ __forceinline__ uint32_t range_word(int lo, int hi, int k) {
  const int a = max(lo - 32 * k, 0), b = min(hi - 32 * k, 32);
  if (a >= b) return 0u;
  const uint32_t hm = b >= 32 ? kAll : (1u << b) - 1u;
  return hm & ~((1u << a) - 1u);
}

struct SweepSmem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  WinMeta meta[kStages][kChunkWins];
  uint32_t dummy[32];
};

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SWEEP_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SWEEP_WAIT;\n"
      "}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
// (producers) poll with a short sleep between attempts: the consumers need the issue slots
__device__ __forceinline__ void bar_wait_backoff(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  for (;;) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
    if (ok) return;
    __nanosleep(100);
  }
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(b))
               : "memory");
}

// row of offset o inside a window (relative to its first row)
__device__ __forceinline__ int row_rel(uint32_t starts, int o) {
  int r = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) r += (int)((starts >> (8 * t)) & 0xFFu) <= o;
  return r;
}

}  // namespace

// dynamic shared memory: [ring: kStages x kChunkWins x kWin int32][hot prefix: hot_words]
__global__ void __launch_bounds__(kSweepThreads, 1) k_sweep(const __grid_constant__ SweepArgs s) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  __shared__ SweepSmem sm;
  int32_t* ring = reinterpret_cast<int32_t*>(s_dyn);
  uint32_t* s_hot = reinterpret_cast<uint32_t*>(s_dyn + kSweepRingBytes);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int hw4 = s.hot_words >> 2;
  uint4* h4 = reinterpret_cast<uint4*>(s_hot);
  griddep_launch();
  for (int i = tid; i < hw4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  __shared__ int32_t s_T[kSmallMax + 2];
  __shared__ int64_t s_B[kSmallMax + 1];
  if (s.n_dense > 0) {
    if (tid < kSmallMax + 2) s_T[tid] = s.classes->T[tid];
    if (tid < kSmallMax + 1) s_B[tid] = s.classes->base[tid];
  }
  if (tid == 0) {
    for (int b = 0; b < kStages; ++b) {
      bar_init(&sm.full[b], 1);
      bar_init(&sm.empty[b], kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  griddep_wait();  // (a programmatic dependent launch: the prologue above ran under the previous kernel's tail)
  const int64_t nchunks = (s.nwin_all + kChunkWins - 1) / kChunkWins;
  const int64_t my_chunks = nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

  if (warp >= kConsumers + kSweepProducers) {
    // ---------------- workers: the dense small region (rows of degree 1..31
    // are one contiguous col_idx range cut at layout time into tasks inside
    // one degree class d): a warp streams a task with 128-bit loads, the next
    // window in flight, and keeps an element when its owner
    // lo_d + (p - base_d) / d is in the frontier bitmap; the targets are OR'ed
    // like the consumers' (same shared copy of the hot prefix)
    const uint32_t hoff = saddr(s_hot);
    const int64_t nw = (int64_t)kSweepWorkers * gridDim.x;
    for (int64_t it = (int64_t)(warp - kConsumers - kSweepProducers) * gridDim.x + blockIdx.x; it < s.n_dense;
         it += nw) {
      const DenseTask dt = s.dense[it];
      const int d = dt.d;
      const int32_t lo = s_T[d + 1];
      const int64_t base = s_B[d];
      const uint32_t rcp = (uint32_t)(0xFFFFFFFFull / (uint32_t)d + 1ull);
      const int64_t a0 = dt.p0 & ~int64_t(3), a1 = dt.p0 + dt.len;
      auto load = [&](int64_t c0) {
        const int64_t p = c0 + lane * 4;
        return p < a1 ? ld_stream4(s.col_idx + p) : make_int4(0, 0, 0, 0);
      };
      int4 cur = load(a0);
      for (int64_t c0 = a0; c0 < a1; c0 += kWin) {
        const int4 nxt = c0 + kWin < a1 ? load(c0 + kWin) : make_int4(0, 0, 0, 0);
        const int64_t p = c0 + lane * 4;
        const int32_t e4[4] = {cur.x, cur.y, cur.z, cur.w};
        int32_t own[4];
        bool in_task[4];
        uint32_t fw[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t pq = p + q;
          const uint32_t rel = (uint32_t)(pq - base);
          own[q] = lo + (d == 1 ? (int32_t)rel : (int32_t)__umulhi(rel, rcp));
          in_task[q] = pq >= dt.p0 && pq < a1;
          fw[q] = in_task[q] ? __ldg(s.front + (own[q] >> 5)) : 0u;  // (read-only during the launch)
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          heavy_or_ok(hoff, (uint32_t)s.hot_words, s.visited, (uint32_t)e4[q], (fw[q] >> (own[q] & 31)) & 1u);
        cur = nxt;
      }
    }
  } else if (warp >= kConsumers) {
    // ---------------- producers: producer warp p takes the CTA's chunks
    // p, p + kProducers, ...; lane j owns window j of a chunk and derives its
    // window info from the side entry and the frontier bitmap.
    const int64_t i0 = warp - kConsumers;
    int st = (int)(i0 % kStages);
    uint32_t ph = (uint32_t)((i0 / kStages) & 1);
    // per window: side entry -> frontier words of its rows -> window_info.
    // The side entry is loaded two iterations ahead and the frontier words
    // (which depend on it) one ahead, so neither latency meets the wait for
    // a free stage; the small-region mask is loaded one ahead
    auto win_of = [&](int64_t i) {
      const int64_t w0 = (blockIdx.x + i * gridDim.x) * kChunkWins;
      return lane < kChunkWins && w0 + lane < s.nwin_all ? w0 + lane : (int64_t)-1;
    };
    auto is_big = [&](int64_t w) { return w >= 0 && w < s.nwin; };
    auto ld_side = [&](int64_t i) {
      const int64_t w = i < my_chunks ? win_of(i) : -1;
      return is_big(w) ? __ldg(s.side + w) : make_uint2(0u, kAll);
    };
    auto ld_front = [&](int64_t i, uint2 sd) {
      const int64_t w = i < my_chunks ? win_of(i) : -1;
      return is_big(w) ? make_uint2(__ldcg(s.front + (sd.x >> 5)), __ldcg(s.front + (sd.x >> 5) + 1))
                       : make_uint2(0u, 0u);
    };
    auto ld_small = [&](int64_t i) {
      const int64_t w = i < my_chunks ? win_of(i) : -1;
      return w >= 0 && w >= s.w_small0 ? __ldcg(s.svmask + (w - s.w_small0)) : make_uint4(0u, 0u, 0u, 0u);
    };
    uint2 sd1 = ld_side(i0), sd2 = ld_side(i0 + kSweepProducers);
    uint2 fw1 = ld_front(i0, sd1);
    uint4 sv1 = ld_small(i0);
    for (int64_t i = i0; i < my_chunks; i += kSweepProducers) {
      const int64_t w = win_of(i);
      const uint2 sd = sd1;
      uint32_t info = window_info(sd, fw1, is_big(w));
      const uint4 sv = sv1;
      sd1 = sd2;
      fw1 = ld_front(i + kSweepProducers, sd1);
      sv1 = ld_small(i + kSweepProducers);
      sd2 = ld_side(i + 2 * kSweepProducers);
      if (s.prefetch > 0 && lane == 0 && i + s.prefetch < my_chunks) {
        // warm L2 with the chunk s.prefetch ahead (whole chunk: its windows'
        // codes are not known yet), so the bulk copy later is an L2 hit
        const int64_t pw = (blockIdx.x + (i + s.prefetch) * gridDim.x) * kChunkWins;
        const int64_t pb = std::min<int64_t>((int64_t)kChunkWins * kWin, s.e_end - pw * kWin) * 4;
        if (pb > 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(s.col_idx + pw * kWin),
                       "r"((uint32_t)((pb + 15) & ~15))
                       : "memory");
      }
      bar_wait_backoff(&sm.empty[st], ph ^ 1u);  // consumers released the stage
      {  // valid-element mask: the ranges of the rows in the frontier, clipped at e_big
        uint32_t vmask[4] = {0u, 0u, 0u, 0u};
        const uint32_t code = info >> 8;
        const int lim = w >= 0 ? (int)std::min<int64_t>(kWin, s.e_big - w * kWin) : 0;
        if (code == 1) {
#pragma unroll
          for (int k = 0; k < 4; ++k) vmask[k] = range_word(0, lim, k);
        } else if (code == 2) {
          int lo = 0;
#pragma unroll
          for (int r = 0; r < 5; ++r) {
            const int hi = r < 4 ? (int)((sd.y >> (8 * r)) & 0xFFu) : 255;  // next row start (0xFF: none)
            const int e = min(min(hi, kWin), lim);
            if ((info >> r) & 1u) {
#pragma unroll
              for (int k = 0; k < 4; ++k) vmask[k] |= range_word(lo, e, k);
            }
            lo = max(lo, min(hi, kWin));
          }
        }
        vmask[0] |= sv.x;  // small-region elements (k_sweep_plan_small)
        vmask[1] |= sv.y;
        vmask[2] |= sv.z;
        vmask[3] |= sv.w;
        const uint32_t any = vmask[0] | vmask[1] | vmask[2] | vmask[3];
        info = (info & 0xFFu) | (any ? 2u << 8 : 0u);
        WinMeta m;
#pragma unroll
        for (int k = 0; k < 4; ++k) m.vmask[k] = vmask[k];
        m.info = info;
        m.pad[0] = m.pad[1] = m.pad[2] = 0u;
        if (lane < kChunkWins) sm.meta[st][lane] = m;
      }
      // one bulk copy per chunk, spanning its first to last window with frontier
      // rows (a bulk copy costs ~0.25 us of TMA issue per SM: few large ones)
      const uint32_t wbytes = w >= 0 ? (uint32_t)((std::min<int64_t>(kWin, s.e_end - w * kWin) * 4 + 15) & ~15) : 0u;
      const uint32_t need = __ballot_sync(kAll, (info >> 8) != 0);
      uint32_t incl = wbytes;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(kAll, incl, o);
        if (lane >= o) incl += t;
      }
      const int lo = need ? __ffs(need) - 1 : 0, hi = need ? 31 - __clz(need) : 0;
      const uint32_t span = __shfl_sync(kAll, incl, hi) - __shfl_sync(kAll, incl, lo) + __shfl_sync(kAll, wbytes, lo);
      __syncwarp();                                                  // every lane's meta store ...
      if (lane == 0) bar_arrive_tx(&sm.full[st], need ? span : 0u);  // ... before the releasing arrive
      if (need && lane == lo)
        bulk_copy(ring + ((size_t)st * kChunkWins + lane) * kWin, s.col_idx + w * kWin, span, &sm.full[st]);
      st += kSweepProducers;  // (kSweepProducers < kStages)
      if (st >= kStages) {
        st -= kStages;
        ph ^= 1u;
      }
    }
  } else {
    // ---------------- consumers: warp c takes windows c*kWinPerWarp .. of each chunk.
    // Nothing is probed: a hot target is OR'ed into the CTA copy, a cold one
    // into the visited bitmap in L2 (red.or, fire and forget); the parents of
    // all the level's new vertices are resolved by k_compact. So no warp ever
    // waits on memory except for its next stage.
    const uint32_t dummy = saddr(&sm.dummy[lane]);  // per-lane sink for masked-off ORs
    const uint32_t hoff = saddr(s_hot);
    const int32_t hv = s.hot_words * 32;            // hot vertices: internal ids < hv
    const int wb = warp * kWinPerWarp;
    int st = 0;
    uint32_t ph = 0;
    for (int64_t i = 0; i < my_chunks; ++i) {
      bar_wait(&sm.full[st], ph);
      // copy this warp's windows (elements + valid nibble) into registers and
      // release the stage at once: the TMA refill of the stage overlaps the
      // ORs below instead of waiting for them
      int4 x[kWinPerWarp];
      uint32_t vm[kWinPerWarp];
      const int32_t* buf = ring + (size_t)st * kChunkWins * kWin;
#pragma unroll
      for (int j = 0; j < kWinPerWarp; ++j) {
        const uint32_t info = sm.meta[st][wb + j].info;
        vm[j] = 0u;
        x[j] = make_int4(0, 0, 0, 0);
        if ((info >> 8) != 0 && !(kSweepDbg & 4)) {  // (warp-uniform) some row of the window is in the frontier
          x[j] = reinterpret_cast<const int4*>(buf + (wb + j) * kWin)[lane];
          vm[j] = (sm.meta[st][wb + j].vmask[lane >> 3] >> (4 * (lane & 7))) & 0xFu;
        }
      }
      __syncwarp();
      if (lane == 0) bar_arrive(&sm.empty[st]);
      if (++st == kStages) {
        st = 0;
        ph ^= 1u;
      }
#pragma unroll
      for (int j = 0; j < kWinPerWarp; ++j) {
        if (!__any_sync(kAll, vm[j] != 0u)) continue;
        const int32_t e4[4] = {x[j].x, x[j].y, x[j].z, x[j].w};
        const int32_t mx = max(max(e4[0], e4[1]), max(e4[2], e4[3]));
        if (__all_sync(kAll, vm[j] == 0xFu && mx < hv)) {
          // whole window valid and hot: one shared OR per element
#if LBFS_SWEEP_HOTCHK
          // skip the OR when the CTA copy already has the bit: the hottest
          // words (the first entries of every hub row) stop taking atomics,
          // which serialise on a shared address
          uint32_t sa[4], bit[4], cw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            asm("shf.l.wrap.b32 %0, 0, 1, %1;" : "=r"(bit[q]) : "r"(e4[q]));
            sa[q] = hoff + (((uint32_t)e4[q] >> 3) & ~3u);
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw[q]) : "r"(sa[q]));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t a = (cw[q] & bit[q]) ? dummy : sa[q];
            if (!(kSweepDbg & 1)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(bit[q]) : "memory");
          }
#elif !defined(LBFS_NO_RUN_MERGE)
          // (adjacent elements in one bitmap word — common in hub rows — take one OR)
          if (!(kSweepDbg & 1))
            heavy_or_hot4(hoff, (uint32_t)e4[0], (uint32_t)e4[1], (uint32_t)e4[2], (uint32_t)e4[3]);
#else
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint32_t bit;
            asm("shf.l.wrap.b32 %0, 0, 1, %1;" : "=r"(bit) : "r"(e4[q]));
            if (!(kSweepDbg & 1))
              asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(hoff + (((uint32_t)e4[q] >> 3) & ~3u)), "r"(bit)
                           : "memory");
          }
#endif
        } else if (!(kSweepDbg & 3) && __all_sync(kAll, vm[j] == 0xFu)) {
          // whole window valid, hot and cold targets: no valid masks to test
#pragma unroll
          for (int q = 0; q < 4; ++q) heavy_or_any(hoff, (uint32_t)s.hot_words, s.visited, (uint32_t)e4[q]);
        } else {
#if LBFS_SWEEP_HOTCHK
          uint32_t sa[4], cw[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const bool ok = (vm[j] >> q) & 1u;
            sa[q] = (ok && e4[q] < hv) ? hoff + (((uint32_t)e4[q] >> 3) & ~3u) : dummy;
            asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw[q]) : "r"(sa[q]));
          }
#endif
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int32_t v = e4[q];
            uint32_t bit;
            asm("shf.l.wrap.b32 %0, 0, 1, %1;" : "=r"(bit) : "r"(v));
            const bool ok = (vm[j] >> q) & 1u;
            const bool hot = v < hv;
#if LBFS_SWEEP_HOTCHK
            const uint32_t sa1 = (cw[q] & bit) ? dummy : sa[q];
#else
            const uint32_t sa1 = (ok && hot) ? hoff + (((uint32_t)v >> 3) & ~3u) : dummy;
#endif
            if (!(kSweepDbg & 1)) asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(sa1), "r"(bit) : "memory");
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.u32 p, %2, 0;\n\t"
                "@p red.relaxed.gpu.global.or.b32 [%0], %1;\n\t}" ::"l"(s.visited + (v >> 5)),
                "r"(bit), "r"((uint32_t)(ok && !hot && !(kSweepDbg & 2)))
                : "memory");
          }
        }
      }
    }
  }

  __syncthreads();
  uint4* row = reinterpret_cast<uint4*>(s.stage) + (size_t)blockIdx.x * (s.stage_words >> 2);
  for (int i = tid; i < hw4; i += blockDim.x) {
    uint4 x = h4[i];
    if (!s.stage_first) {
      const uint4 y = __ldcg(row + i);
      x.x |= y.x, x.y |= y.y, x.z |= y.z, x.w |= y.w;
    }
    __stcg(row + i, x);
  }
}

}  // namespace lbfs
