// Top-down BFS on sm_100a: the hot path of the reference's run_bfs
// (traversal.py:413-422 -> bfs_serial / bfs_parallel_naive / _bitmap_bfs,
// traversal.py:80-389).
//
//   K4 k_init_seed       PredecessorArray fill + Bitmap clear + root seed in
//                        one launch (traversal.py:42-46, 135-139, 343-347;
//                        the partitioned path keeps k_init + k_seed)
//   K1 k_expand<Mode, bins>  frontier expansion over CSR by one persistent
//                        CTA per SM, one launch per non-empty bin (slice
//                        items + raw queues share one after a queue level):
//                        - slice items (rows of deg >= kCtaMin cut on window
//                          boundaries into <= kChunk / qchunk elements; after
//                          a queue or cluster level also the rows with
//                          32 <= deg < kCtaMin): a warp streams its slices in
//                          groups of D 128-element windows, 128-bit loads,
//                          the next group in flight;
//                        - warp slices (32 <= deg < kCtaMin after a bitmap
//                          level): one slice per row, same streamer;
//                        - group items / raw small queue (deg < 32): a warp
//                          takes up to 32 vertices and walks their
//                          concatenated rows; groups of one degree class map
//                          elements to rows in closed form (no row_ptr read);
//                        - dense small region: the rows of degree 1..31 as
//                          one stream filtered by the frontier bitmap.
//                        Replaces _frontier_neighbors + the 16-lane Listing-1
//                        gather (traversal.py:107-119, 297-332). Heavy levels
//                        also use k_sweep (sweep.cu), small levels
//                        k_cluster_levels (cluster.cu).
//   K2 probe + settle    visited test: words of the hot bitmap prefix from a
//                        per-SM shared-memory copy, the rest from L2. Bitmap
//                        mode settles a clear bit without waiting: red.or on
//                        the bitmap + the parent into pred_int (any
//                        equal-level parent is valid, traversal.py:145-147);
//                        queue mode elects one winner with atomicOr; heavy
//                        mode ORs blindly (no probe, no parent: k_resolve
//                        finds the parents afterwards). Replaces the
//                        unsynchronised OR + negative marks + restoration
//                        pass (traversal.py:175-279).
//   K3 next frontier     queue mode: warp-aggregated appends by the winners
//                        (small queue + slice items); bitmap / heavy mode:
//                        k_compact turns the new visited bits into the next
//                        frontier bitmap, list, group items and slices with
//                        block-aggregated appends and writes the levels.
//                        Replaces the np.unique merge / nonzero-word scans
//                        (traversal.py:157-158, 168-172, 366-384).
//   K5 BfsEngine::run    level driver (the while loops traversal.py:90,152,366):
//                        mapped-memory mailbox per level, k_publish or the
//                        cluster kernel as the publisher
//   K6 Counters          LayerStats(input, edges, discovered) per level
//                        (traversal.py:66-70, 100, 159, 383)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "bfs_engine.cuh"

namespace lbfs {

constexpr unsigned kFull = 0xFFFFFFFFu;
// kQueueDirect: queue mode without the visited pre-probe
// kHeavy: bitmap mode for the heavy levels (most of the graph's edges in one
// level): every target is OR'ed blindly — hot-prefix targets into the CTA's
// zeroed shared copy (k_merge_hot folds the copies into the visited bitmap),
// the rest into visited in L2 — with no probe and no parent (k_resolve gives
// the level's new vertices their parents on a side stream).
// (enum Mode: bfs_engine.cuh)
#ifndef LBFS_CHECKS
#define LBFS_CHECKS 0  // debug builds: bounds checks that trap with a location
#endif
#if LBFS_CHECKS
#define LBFS_DCHECK(cond, what)                                                                   \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("[lbfs check] %s failed at %s:%d (block %d thread %d)\n", what, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define LBFS_DCHECK(cond, what) \
  do {                          \
  } while (0)
#endif

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
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void red_or(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
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

struct Hot {  // shared-memory copy of the visited words [0, words)
  uint32_t* s;
  uint32_t base;  // shared-window address of s
  int32_t words;
};

// Per-warp shared scratch for the group walks.
struct WarpScratch {
  int32_t off[33];
  int32_t vert[32];
  int64_t start[32];
};

__device__ __forceinline__ bool bit_clear(uint32_t word, int32_t v) { return ((word >> (v & 31)) & 1u) == 0; }

// (single-partition runs only: ids are local == global)
// Queue mode (warp-collective), a batch of K candidates per lane: the K
// atomicOr elections are in flight together; winners write level + pred and
// are appended to the next level's bins with one atomic per bin per warp for
// the whole batch (a packed warp scan of the per-lane counts). Hub winners
// (rare) also emit kChunk slices.
template <int K, typename ParFn>
__device__ __forceinline__ void settle_queue(const LevelArgs& a, const int32_t (&nb)[K], uint32_t cmask, ParFn par,
                                             int lane, Acc& acc) {
  uint32_t old[K];
#pragma unroll
  for (int k = 0; k < K; ++k)
    old[k] = ((cmask >> k) & 1u) ? atomicOr(a.visited + (nb[k] >> 5), 1u << (nb[k] & 31)) : kFull;
  uint32_t win = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) win |= (((old[k] >> (nb[k] & 31)) & 1u) ^ 1u) << k;
  if (!__any_sync(kFull, win != 0)) return;
  int64_t st[K];
  int32_t deg[K];
  uint32_t ns = 0, nw = 0;
  bool hub = false;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    st[k] = 0;
    deg[k] = 0;
    if ((win >> k) & 1u) {
      const int32_t v = nb[k];
      st[k] = a.row_ptr[v];
      deg[k] = (int32_t)(a.row_ptr[v + 1] - st[k]);
      ns += (v >= a.t_warp && v < a.t_nz);
      nw += (v >= a.t_hub && v < a.t_warp);
      hub |= v < a.t_hub;
    }
  }
  // exclusive offsets of this lane's small (low half) and warp (high half) appends
  uint32_t incl = ns | (nw << 16);
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t tot = __shfl_sync(kFull, incl, 31);
  unsigned long long bs = 0, bw = 0;
  if (lane == 0) {
    if (tot & 0xFFFFu) bs = atomicAdd(&a.next_cnt->bin[kBinSmall], (unsigned long long)(tot & 0xFFFFu));
    if (tot >> 16) bw = atomicAdd(&a.next_cnt->bin[kBinWarp], (unsigned long long)(tot >> 16));
  }
  const uint32_t excl = incl - (ns | (nw << 16));
  unsigned long long os = __shfl_sync(kFull, bs, 0) + (excl & 0xFFFFu);
  unsigned long long ow = __shfl_sync(kFull, bw, 0) + (excl >> 16);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (!((win >> k) & 1u)) continue;
    const int32_t v = nb[k];
    atomicOr(a.prev + (v >> 5), 1u << (v & 31));  // keep bitmap-mode compaction exact
    a.level_int[v] = a.next_level;                 // internal order; k_finalize writes the outputs
    a.pred_int[v] = par(k);                        // parents travel as original ids
    if (v >= a.t_warp && v < a.t_nz) a.next_small[os++] = v;
    if (v >= a.t_hub && v < a.t_warp) a.next_warp[ow++] = v;
    acc.disc += 1;
    acc.edges += (unsigned long long)deg[k];
  }
  if (!__any_sync(kFull, hub)) return;
  // rows below t_hub become slice items (cut on window boundaries): one
  // reservation per warp for the items of all K candidates (each reservation
  // is an L2 atomic round trip on the level's critical chain)
  int items[K];
  int32_t vo[K];
  int mine = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool w = ((win >> k) & 1u) && nb[k] < a.t_hub;
    items[k] = !w ? 0 : a.align_items ? slice_items(st[k], deg[k], a.qchunk) : (deg[k] + a.qchunk - 1) / a.qchunk;
    vo[k] = w ? __ldg(a.new2old + nb[k]) : 0;
    mine += items[k];
  }
  int inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += t;
  }
  const int total = __shfl_sync(kFull, inc, 31);
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(&a.next_cnt->bin[kBinCta], (unsigned long long)total);
  base = __shfl_sync(kFull, base, 31) + (unsigned long long)(inc - mine);
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int j = 0; j < items[k]; ++j)
      a.next_cta[base++] = a.align_items ? slice_item(st[k], deg[k], a.qchunk, j, vo[k])
                                         : CtaItem{st[k] + (int64_t)j * a.qchunk, min(a.qchunk, deg[k] - j * a.qchunk), vo[k]};
}

// Probe a batch of K neighbours. Words of the hot prefix come from the
// shared copy (a random 32-lane gather costs a few bank cycles there versus
// ~32 L1 wavefronts); cold words use L1-cached loads. All K loads are issued
// before any of them is consumed.
//
// Bitmap mode settles a clear bit without waiting on memory: any lane whose
// view (shared copy, L1 line or L2 word — all loaded after the level
// started) shows v unvisited may record its parent, since every such parent
// is one level up (the benign race of bfs_parallel_naive,
// traversal.py:145-147). Lanes hitting the same bitmap word elect one
// writer: one red.or to the bitmap and one OR into the shared copy per word
// per warp step; each lane stores its parent (original id) to pred_int[v].

// Heavy levels: blind OR of target v (when ok != 0): into the CTA's shared
// copy when its word is below hot_words, else into visited in L2. Predicated,
// no branch.
__device__ __forceinline__ void heavy_or(const Hot& h, const uint32_t* visited, uint32_t v, uint32_t ok,
                                         uint32_t hot_words) {
  asm volatile(
      "{\n\t"
      ".reg .pred pk, ph, pc;\n\t"
      ".reg .u32 wi, sa, bit;\n\t"
      ".reg .u64 ga;\n\t"
      "shr.u32 wi, %0, 5;\n\t"
      "shf.l.wrap.b32 bit, 0, 1, %0;\n\t"
      "setp.ne.u32 pk, %1, 0;\n\t"
      "setp.lt.and.u32 ph, wi, %2, pk;\n\t"
      "setp.ge.and.u32 pc, wi, %2, pk;\n\t"
      "shl.b32 sa, wi, 2;\n\t"
      "add.u32 sa, sa, %3;\n\t"
      "mad.wide.u32 ga, wi, 4, %4;\n\t"
      "@ph red.shared.or.b32 [sa], bit;\n\t"
      "@pc red.relaxed.gpu.global.or.b32 [ga], bit;\n\t"
      "}" ::"r"(v),
      "r"(ok), "r"(hot_words), "r"(h.base), "l"(visited)
      : "memory");
}
// ... every lane's target known valid (a full interior window)
__device__ __forceinline__ void heavy_or_full(const Hot& h, const uint32_t* visited, uint32_t v) {
  asm volatile(
      "{\n\t"
      ".reg .pred ph;\n\t"
      ".reg .u32 wi, sa, bit;\n\t"
      ".reg .u64 ga;\n\t"
      "shr.u32 wi, %0, 5;\n\t"
      "shf.l.wrap.b32 bit, 0, 1, %0;\n\t"
      "setp.lt.u32 ph, wi, %1;\n\t"
      "shl.b32 sa, wi, 2;\n\t"
      "add.u32 sa, sa, %2;\n\t"
      "mad.wide.u32 ga, wi, 4, %3;\n\t"
      "@ph red.shared.or.b32 [sa], bit;\n\t"
      "@!ph red.relaxed.gpu.global.or.b32 [ga], bit;\n\t"
      "}" ::"r"(v),
      "r"((uint32_t)h.words), "r"(h.base), "l"(visited)
      : "memory");
}
// ... target known to lie in the hot prefix
__device__ __forceinline__ void heavy_or_hot(const Hot& h, uint32_t v, uint32_t ok) {
  asm volatile(
      "{\n\t"
      ".reg .pred pk;\n\t"
      ".reg .u32 sa, bit;\n\t"
      "shf.l.wrap.b32 bit, 0, 1, %0;\n\t"
      "setp.ne.u32 pk, %1, 0;\n\t"
      "shr.u32 sa, %0, 3;\n\t"
      "and.b32 sa, sa, 0xfffffffc;\n\t"
      "add.u32 sa, sa, %2;\n\t"
      "@pk red.shared.or.b32 [sa], bit;\n\t"
      "}" ::"r"(v),
      "r"(ok), "r"(h.base)
      : "memory");
}
__device__ __forceinline__ void heavy_or_hot_full(const Hot& h, uint32_t v) {
  asm volatile(
      "{\n\t"
      ".reg .u32 sa, bit;\n\t"
      "shf.l.wrap.b32 bit, 0, 1, %0;\n\t"
      "shr.u32 sa, %0, 3;\n\t"
      "and.b32 sa, sa, 0xfffffffc;\n\t"
      "add.u32 sa, sa, %1;\n\t"
      "red.shared.or.b32 [sa], bit;\n\t"
      "}" ::"r"(v),
      "r"(h.base)
      : "memory");
}

// Visited word of v's bitmap word wi: from the shared copy when wi is in the
// hot prefix, else from L2 — two predicated loads, no branch, no generic
// addressing. (Not through L1: within one k_bfs launch an L1 line may date
// from an earlier level, and an old "unvisited" would record a parent two
// levels up; the L1 hit rate of these probes was 1-8% anyway.)
__device__ __forceinline__ uint32_t probe_word(const Hot& h, const uint32_t* visited, int32_t wi) {
  uint32_t w;
  asm("{\n\t.reg .pred p;\n\t"
      "setp.lt.s32 p, %1, %2;\n\t"
      "@p ld.shared.u32 %0, [%3];\n\t"
      "@!p ld.global.cg.u32 %0, [%4];\n\t}"
      : "=r"(w)
      : "r"(wi), "r"(h.words), "r"(h.base + 4u * (uint32_t)wi), "l"(visited + wi));
  return w;
}

// Bitmap mode, candidates in cmask: runs of candidates in one bitmap word
// (consecutive elements of a lane come from sorted rows) are merged into a
// single red.or + shared OR; each candidate stores its parent.
template <int K, typename ParFn>
__device__ __forceinline__ void settle_bitmap(const LevelArgs& a, const Hot& h, const int32_t (&nb)[K],
                                              uint32_t cmask, ParFn par) {
  int32_t run_w = -1;
  uint32_t run_bits = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (!((cmask >> k) & 1u)) continue;
    const int32_t v = nb[k];
    const int32_t wi = v >> 5;
    LBFS_DCHECK(v >= 0 && (int64_t)v < a.chk_n, "settle_bitmap target id");
    if (wi != run_w) {
      if (run_bits) {
        red_or(a.visited + run_w, run_bits);
        if (run_w < h.words) atomicOr(h.s + run_w, run_bits);
      }
      run_w = wi;
      run_bits = 0;
    }
    run_bits |= 1u << (v & 31);
    // partitioned: a neighbour owned by another rank is only marked; its
    // owner resolves the parent after the exchange (partition.cu)
    if (part_owned(v, a.part_log, a.part_rank)) a.pred_int[part_local(v, a.part_log)] = par(k);
    if (a.dbg) atomicAdd(a.dbg + (wi < h.words ? 0 : 1), 1ull);  // LBFS_COUNT only
  }
  red_or(a.visited + run_w, run_bits);
  if (run_w < h.words) atomicOr(h.s + run_w, run_bits);
}

// Probe a batch of K neighbours (elements outside okmask must hold a valid
// id, e.g. 0). All K loads are issued before any is consumed. Bitmap mode
// settles clear bits without waiting on memory: any lane whose view (shared
// copy, L1 line or L2 word — all loaded after the level started) shows v
// unvisited may record its parent, since every such parent is one level up
// (the benign race of bfs_parallel_naive, traversal.py:145-147). Queue mode
// elects one winner per vertex with atomicOr.
// Where a batch's visited words are known to lie (warp-uniform): sorted
// interior chunks of a row are classified once by their first/last element.
enum Where : int { kMixed = 0, kAllHot = 1, kAllCold = 2 };

// Candidate mask of a batch: bit k set when nb[k] (valid per okmask) reads
// as unvisited.
template <int M, int K, int W = kMixed>
__device__ __forceinline__ uint32_t probe_mask(const LevelArgs& a, const Hot& h, const int32_t (&nb)[K],
                                               uint32_t okmask) {
  if constexpr (M == kQueueDirect) return okmask;
  uint32_t cmask = 0;
  if constexpr (M == kHeavy) {
    // hot: one red.shared.or into the CTA copy, cold: one red.or into visited
    // in L2; nothing waits on memory and no parent is recorded (k_resolve
    // gives every new vertex of a heavy level its parent). Branch-free: the
    // heavy kernels are issue-bound (ncu: 81% issue slots busy with a branchy
    // hot/cold split, ~22 instructions per element), so each element is a
    // word index, a bit, two predicates and two predicated reductions.
#pragma unroll
    for (int k = 0; k < K; ++k) {
      LBFS_DCHECK(!((okmask >> k) & 1u) || (nb[k] >= 0 && (int64_t)nb[k] < a.chk_n), "heavy probe target id");
      if constexpr (W == kAllHot)
        heavy_or_hot(h, (uint32_t)nb[k], okmask & (1u << k));
      else
        heavy_or(h, a.visited, (uint32_t)nb[k], okmask & (1u << k), W == kAllCold ? 0u : (uint32_t)h.words);
    }
    return 0u;
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    uint32_t w;
    if constexpr (W == kAllHot)
#ifdef LBFS_HOT_GENERIC
      w = h.s[nb[k] >> 5];
#else
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(h.base + 4u * (uint32_t)(nb[k] >> 5)));
#endif
    else if constexpr (W == kAllCold)
      w = __ldcg(a.visited + (nb[k] >> 5));
    else
      w = probe_word(h, a.visited, nb[k] >> 5);
    cmask |= ((~w >> (nb[k] & 31)) & 1u) << k;
  }
  return cmask & okmask;
}

// Settle the candidates of a batch (queue modes: warp-collective).
template <int M, int K, typename ParFn>
__device__ __forceinline__ void settle(const LevelArgs& a, const Hot& h, const int32_t (&nb)[K], uint32_t cmask,
                                       ParFn par, int lane, Acc& acc) {
  if constexpr (M == kBitmapOut || M == kHeavy) {
    if (cmask) settle_bitmap<K>(a, h, nb, cmask, par);
  } else {
    settle_queue<K>(a, nb, cmask, par, lane, acc);
  }
}

template <int M, int K, typename ParFn, int W = kMixed>
__device__ __forceinline__ void probe_batch(const LevelArgs& a, const Hot& h, const int32_t (&nb)[K],
                                            uint32_t okmask, ParFn par, int lane, Acc& acc) {
  settle<M, K>(a, h, nb, probe_mask<M, K, W>(a, h, nb, okmask), par, lane, acc);
}

template <int M>
__device__ __forceinline__ void flush_acc(const LevelArgs& a, Acc& acc) {
  if constexpr (M == kQueueOut || M == kQueueDirect) {
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

// ---------------------------------------------------------------- K1 pieces
// degree class of a small-region internal id: the d with T[d+1] <= v < T[d]
__device__ __forceinline__ int degree_class(const int32_t* T, int32_t v) {
  int d = 1;  // largest d in [1, kSmallMax-1] with T[d] > v (T non-increasing)
#pragma unroll
  for (int step = 16; step; step >>= 1)
    if (d + step <= kSmallMax - 1 && T[d + step] > v) d += step;
  return d;
}

__device__ __forceinline__ uint32_t range_mask(int64_t base_v, int64_t lo, int64_t hi) {
  // bits b with lo <= base_v + b < hi
  const int64_t a = std::max<int64_t>(lo - base_v, 0), b = std::min<int64_t>(hi - base_v, 32);
  if (a >= b) return 0u;
  const uint32_t hi_m = (b >= 32) ? kFull : ((1u << b) - 1u);
  const uint32_t lo_m = (a >= 32) ? kFull : ((1u << a) - 1u);
  return hi_m & ~lo_m;
}

// A warp expands elements [elo, ehi) of the concatenated rows of up to 32
// vertices (lanes [0, n) own one each): one row_ptr round trip, a degree
// scan, then 128-element windows in which each lane finds its element's
// owner by binary search over the group's offsets.
template <int M>
__device__ __forceinline__ void expand_group(const LevelArgs& a, const Hot& h, int n, int32_t u, int dcls, int elo,
                                             int ehi, const int32_t* T, const int64_t* B, int lane, WarpScratch& ws,
                                             Acc& acc) {
  int64_t st = 0;
  int32_t d = 0, uo = 0;
  if (lane < n) {
    if (dcls > 0) {  // small region: row from the degree-class table, no row_ptr read
      d = dcls;
      st = B[dcls] + (int64_t)(u - T[dcls + 1]) * dcls;
    } else {
      st = a.row_ptr[u];
      d = (int32_t)(a.row_ptr[u + 1] - st);
    }
    uo = __ldg(a.new2old + u);
  }
  int incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += t;
  }
  const int total = __shfl_sync(kFull, incl, 31);
  const int end = min(ehi, total);
  __syncwarp();
  ws.off[lane] = incl - d;
  ws.start[lane] = st - (incl - d);
  ws.vert[lane] = uo;
  __syncwarp();
  // software-pipelined 128-element windows: window i+1's col_idx loads are
  // in flight while window i is probed. The owner of element e is found by a
  // binary search over the n row offsets: ceil(log2 n) steps (none for a
  // single row, e.g. a warp-bin queue entry); entries >= n hold the total, so
  // the search never leaves [0, n)
  const int top = n > 1 ? 1 << (31 - __clz(n - 1)) : 0;  // largest power of two < n
  auto load_win = [&](int e0, int32_t (&nb)[4], int32_t (&par)[4]) -> uint32_t {
    uint32_t okm = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * 32 + lane;
      const bool ok = e < end;
      okm |= (uint32_t)ok << k;
      int lo = 0;
      for (int step = top; step; step >>= 1)
        if (ws.off[lo + step] <= e) lo += step;
      LBFS_DCHECK(!ok || (ws.start[lo] + e >= 0 && ws.start[lo] + e < a.chk_nnz), "expand_group element");
      nb[k] = ok ? ld_stream(a.col_idx + ws.start[lo] + e) : 0;
      par[k] = ws.vert[lo];
    }
    return okm;
  };
  int32_t nbA[4], parA[4], nbB[4], parB[4];
  uint32_t okA = elo < end ? load_win(elo, nbA, parA) : 0u;
  for (int e0 = elo; e0 < end; e0 += 128) {
    const uint32_t okB = (e0 + 128 < end) ? load_win(e0 + 128, nbB, parB) : 0u;
    probe_batch<M, 4>(a, h, nbA, okA, [&](int k) { return parA[k]; }, lane, acc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      nbA[k] = nbB[k];
      parA[k] = parB[k];
    }
    okA = okB;
  }
  __syncwarp();
}

// Elements [elo, ehi) of a group whose vertices all have degree d (lanes
// [0, n) valid): the rows of class d are contiguous from T/base, so element
// e belongs to lane e / d at offset e % d — no row_ptr read, no search.
template <int M>
__device__ __forceinline__ void expand_class_group(const LevelArgs& a, const Hot& h, int n, int32_t v, int d,
                                                   int elo, int ehi, const int32_t* T, const int64_t* B, int lane,
                                                   Acc& acc) {
  const int32_t roff = (lane < n) ? (v - T[d + 1]) * d : 0;
  const int32_t vo = (lane < n) ? __ldg(a.new2old + v) : 0;
  const int32_t* rows = a.col_idx + B[d];
  const uint32_t rcp = (uint32_t)(0xFFFFFFFFull / (uint32_t)d + 1ull);  // e / d for e < 2^27, d >= 2
  const int end = min(ehi, n * d);
  auto load_win = [&](int e0, int32_t (&nb)[4], int32_t (&par)[4]) -> uint32_t {
    uint32_t okm = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = e0 + k * 32 + lane;
      const bool ok = e < end;
      okm |= (uint32_t)ok << k;
      const int q = !ok ? 0 : (d == 1 ? e : (int)__umulhi((uint32_t)e, rcp));
      const int32_t ro = __shfl_sync(kFull, roff, q);
      par[k] = __shfl_sync(kFull, vo, q);
      nb[k] = ok ? ld_stream(rows + ro + (e - q * d)) : 0;
    }
    return okm;
  };
  int32_t nbA[4], parA[4], nbB[4], parB[4];
  uint32_t okA = elo < end ? load_win(elo, nbA, parA) : 0u;
  for (int e0 = elo; e0 < end; e0 += 128) {
    const uint32_t okB = (e0 + 128 < end) ? load_win(e0 + 128, nbB, parB) : 0u;
    probe_batch<M, 4>(a, h, nbA, okA, [&](int k) { return parA[k]; }, lane, acc);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      nbA[k] = nbB[k];
      parA[k] = parB[k];
    }
    okA = okB;
  }
}

// Elements [elo, ehi) of a group of up to 32 vertices (lanes [0, n)):
// closed-form walk when all lie in one small-region degree class (the common
// case with degree-ordered ids), generic walk otherwise.
template <int M>
__device__ __forceinline__ void expand_range(const LevelArgs& a, const Hot& h, int n, int32_t v, int elo, int ehi,
                                             const int32_t* T, const int64_t* B, int lane, WarpScratch& ws,
                                             Acc& acc) {
  const bool small = (lane < n) && v >= a.t_warp && v < a.t_nz;
  const int d = small ? degree_class(T, v) : 0;
  const int d0 = __shfl_sync(kFull, d, 0);
  if (d0 > 0 && __all_sync(kFull, lane >= n || d == d0))
    expand_class_group<M>(a, h, n, v, d0, elo, ehi, T, B, lane, acc);
  else
    expand_group<M>(a, h, n, v, d, elo, ehi, T, B, lane, ws, acc);
}

// Slice descriptors through L2 (k_levels rewrites a queue buffer every other
// level within one launch; L1 is not coherent).
__device__ __forceinline__ CtaItem ld_item(const CtaItem* p) {
  const int4 r = __ldcg(reinterpret_cast<const int4*>(p));
  CtaItem c;
  c.start = (int64_t)(((uint64_t)(uint32_t)r.y << 32) | (uint32_t)r.x);
  c.len = r.z;
  c.u = r.w;
  return c;
}

// A warp walks row slices (grid-stride over items) in groups of D
// 128-element windows, one 128-bit load per lane per window; the next
// group's D loads are issued before the current group is probed, so a warp
// keeps 2 x D x 512 B in flight (D = 4 for heavy levels, whose per-element
// work is light; 2 where the settle path needs the registers).
template <int M>
constexpr int slice_depth() { return M == kHeavy || M == kQueueOut ? 4 : 2; }

template <int M, typename Fetch>
__device__ __forceinline__ void stream_slices_f(const LevelArgs& a, const Hot& h, Fetch fetch, int64_t n64,
                                                int64_t gwarp, int64_t nwarps64, int lane, Acc& acc) {
  constexpr int D = slice_depth<M>();
  if (gwarp >= n64) return;
  // (item counts are bounded by the item buffers: nnz / 128 + hubs < 2^31)
  const int32_t n = (int32_t)n64, nwarps = (int32_t)nwarps64;
  int32_t it = (int32_t)gwarp;
  CtaItem cur = fetch(it);
  // the descriptor after cur is loaded one row ahead, so a row switch never
  // waits on it before issuing the row's first col_idx load
  CtaItem nxt = it + nwarps < n ? fetch(it + nwarps) : CtaItem{0, 0, 0};
  // A slice in window coordinates: lp points at this lane's first element of
  // the slice's first 128-bit-aligned window; mis = start & 3 elements of that
  // window precede the slice, which ends at offset mis + len; span = the
  // aligned extent. (32-bit offsets from one 64-bit pointer: the loop's
  // address and bounds arithmetic stays out of 64-bit registers.)
  const int32_t* lp = a.col_idx + (cur.start & ~int64_t(3)) + lane * 4;
  int32_t mis = (int32_t)(cur.start & 3);
  int32_t span = (mis + cur.len + 3) & ~3;
  int32_t w = 0;  // offset of the next group's first window
  auto load_group = [&](const int32_t* q, int32_t w0, int32_t sp, int4 (&x)[D]) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int32_t o = w0 + d * 128;
      LBFS_DCHECK(!(o + lane * 4 < sp) || (q + o >= a.col_idx && q + o + 4 <= a.col_idx + a.chk_nnz + 8), "slice load");
      x[d] = o + lane * 4 < sp ? ld_stream4(q + o) : make_int4(0, 0, 0, 0);
    }
  };
  int4 xa[D];
  load_group(lp, 0, span, xa);
  while (true) {
    const int32_t g_w = w, g_lo = mis, g_hi = mis + cur.len;  // this group's slice bounds
    const int32_t pu = cur.u;
    w += D * 128;
    bool more = true;
    if (w >= span) {
      it += nwarps;
      if (it < n) {
        cur = nxt;
        if (it + nwarps < n) nxt = fetch(it + nwarps);
        lp = a.col_idx + (cur.start & ~int64_t(3)) + lane * 4;
        mis = (int32_t)(cur.start & 3);
        span = (mis + cur.len + 3) & ~3;
        w = 0;
      } else {
        more = false;
      }
    }
    int4 xb[D];
    if (more) {
      load_group(lp, w, span, xb);
    } else {
#pragma unroll
      for (int d = 0; d < D; ++d) xb[d] = make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int32_t cw = g_w + d * 128;  // the window's offset
      if (cw >= g_hi) break;             // (warp-uniform) past the slice
      if constexpr (M == kHeavy) {
        // (warp-uniform) a window inside the slice: no valid masks; a slice is
        // part of one sorted row, so lane 31's last element is the window's
        // largest id and tells whether every target is in the hot prefix
        if (cw >= g_lo && cw + 128 <= g_hi) {
          if (a.dbg) atomicAdd(a.dbg + 2, 4ull);  // LBFS_COUNT: slice elements
          const uint32_t last = __shfl_sync(kFull, (uint32_t)xa[d].w, 31);
          if ((last >> 5) < (uint32_t)h.words) {
#ifdef LBFS_NO_RUN_MERGE
            heavy_or_hot_full(h, (uint32_t)xa[d].x);
            heavy_or_hot_full(h, (uint32_t)xa[d].y);
            heavy_or_hot_full(h, (uint32_t)xa[d].z);
            heavy_or_hot_full(h, (uint32_t)xa[d].w);
#else
            heavy_or_hot4(h.base, (uint32_t)xa[d].x, (uint32_t)xa[d].y, (uint32_t)xa[d].z, (uint32_t)xa[d].w);
#endif
          } else {
            heavy_or_full(h, a.visited, (uint32_t)xa[d].x);
            heavy_or_full(h, a.visited, (uint32_t)xa[d].y);
            heavy_or_full(h, a.visited, (uint32_t)xa[d].z);
            heavy_or_full(h, a.visited, (uint32_t)xa[d].w);
          }
          continue;
        }
      }
      int32_t nb[4] = {xa[d].x, xa[d].y, xa[d].z, xa[d].w};
      const int lo = g_lo - cw - lane * 4, hi = g_hi - cw - lane * 4;
      uint32_t okm = 0xFu;
      if (lo > 0 || hi < 4) {  // first/last window of a slice
        okm = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const bool ok = q >= lo && q < hi;
          okm |= (uint32_t)ok << q;
          nb[q] = ok ? nb[q] : 0;
        }
      }
      if (a.dbg) atomicAdd(a.dbg + 2, (unsigned long long)__popc(okm));  // LBFS_COUNT: slice elements
      probe_batch<M, 4>(a, h, nb, okm, [&](int) { return pu; }, lane, acc);
    }
    if (!more) break;
#pragma unroll
    for (int d = 0; d < D; ++d) xa[d] = xb[d];
  }
}

template <int M>
__device__ __forceinline__ void stream_slices(const LevelArgs& a, const Hot& h, const CtaItem* items, int64_t n,
                                              int64_t gwarp, int64_t nwarps, int lane, Acc& acc) {
  stream_slices_f<M>(a, h, [&](int64_t i) { return ld_item(items + i); }, n, gwarp, nwarps, lane, acc);
}

// Warp-bin rows of a queue-mode frontier (raw vertex ids) streamed like
// slices: the row of queue entry i is [row_ptr[v], row_ptr[v+1]) with parent
// new2old[v], fetched one row ahead (pipelined, unlike one expand_range call
// per row).
template <int M>
__device__ __forceinline__ void stream_queue_rows(const LevelArgs& a, const Hot& h, const int32_t* q, int64_t n,
                                                  int64_t gwarp, int64_t nwarps, int lane, Acc& acc) {
  stream_slices_f<M>(
      a, h,
      [&](int64_t i) {
        const int32_t v = __ldcg(q + i);
        const int64_t st = __ldg(a.row_ptr + v);
        return CtaItem{st, (int32_t)(__ldg(a.row_ptr + v + 1) - st), __ldg(a.new2old + v)};
      },
      n, gwarp, nwarps, lane, acc);
}

// Static shared memory of an expansion CTA (kExpandWarps warps); the
// dynamic part is the snapshot of the visited prefix.
struct ExpandSmem {
  uint64_t hot_bar;                         // hot snapshot copies
  WarpScratch ws[kExpandWarps];
  int32_t T[kSmallMax + 2];
  int64_t B[kSmallMax + 1];
  uint32_t hot_issued;  // snapshot copies issued so far (thread 0 only issues)
};

__device__ __forceinline__ void expand_init(ExpandSmem& s, const LevelArgs& a) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    mbar_init(&s.hot_bar, 1);
    s.hot_issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kSmallMax + 2) s.T[tid] = a.classes->T[tid];
  if (tid < kSmallMax + 1) s.B[tid] = a.classes->base[tid];
  __syncthreads();
}

// (thread 0) wait until the last snapshot copy has landed
__device__ __forceinline__ void hot_wait_last(ExpandSmem& s) {
  if (s.hot_issued) mbar_wait(&s.hot_bar, (s.hot_issued - 1) & 1u);
}
// (thread 0) issue a snapshot copy of the visited prefix
__device__ __forceinline__ void hot_issue(ExpandSmem& s, const Hot& h, const uint32_t* visited) {
  const uint32_t bytes = (uint32_t)h.words * 4u;  // multiple of 16 by construction
  mbar_expect_tx(&s.hot_bar, bytes);
  bulk_g2s(h.s, visited, bytes, &s.hot_bar);
  ++s.hot_issued;
}
// (all threads) load the snapshot and wait for it
__device__ __forceinline__ void hot_load(ExpandSmem& s, const Hot& h, const uint32_t* visited) {
  if (h.words <= 0) return;
  __syncthreads();  // nobody still reads the old snapshot
  if (threadIdx.x == 0) {
    hot_wait_last(s);
    hot_issue(s, h, visited);
  }
  __syncthreads();
  mbar_wait(&s.hot_bar, (s.hot_issued - 1) & 1u);
}
// (all threads) no snapshot copy in flight (before reusing or leaving the smem)
__device__ __forceinline__ void hot_drain(ExpandSmem& s) {
  if (threadIdx.x == 0) hot_wait_last(s);
  __syncthreads();
}

// The expansion of one level's frontier by one persistent CTA per SM,
// bins selected by kPhases.
template <int M, int kPhases>
__device__ __forceinline__ void expand_phases(const LevelArgs& a, const Frontier& f, ExpandSmem& s, const Hot& h,
                                              Acc& acc) {
  constexpr int phases = kPhases;
  const int tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
  // warp ids interleave the SMs so that the first work units of every phase
  // land on different SMs
  const int64_t gwarp = (int64_t)wib * gridDim.x + blockIdx.x;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  WarpScratch& ws = s.ws[wib];
  const int32_t* s_T = s.T;
  const int64_t* s_B = s.B;

  // ---- phase 1: hub slices (deg >= kCtaMin), one kChunk slice per warp step,
  // 128-bit loads with the next chunk in flight. (Round 1 staged them through
  // a per-warp cp.async.bulk ring; that variant failed certification
  // intermittently — DESIGN.md §5 — and is gone.)
  if (phases & 1) stream_slices<M>(a, h, f.cta, f.n_cta, gwarp, nwarps, lane, acc);

  // ---- phase 2a: warp-bin rows (32 <= deg < kCtaMin), one slice each -----
  if (phases & 16) stream_slices<M>(a, h, f.wslice, f.n_wslice, gwarp, nwarps, lane, acc);

  // ---- phase 2: non-hub frontier as balanced group items -----------------
  for (int64_t it = gwarp; (phases & 2) && it < f.n_items; it += nwarps) {
    GroupItem gi;
    {  // through L2: written within the same launch by k_bfs (24-byte items: 8-byte loads)
      const int2* r = reinterpret_cast<const int2*>(f.items + it);
      const int2 r0 = __ldcg(r), r1 = __ldcg(r + 1), r2 = __ldcg(r + 2);
      gi.list_start = (int64_t)(((uint64_t)(uint32_t)r0.y << 32) | (uint32_t)r0.x);
      gi.count = r1.x;
      gi.elo = r1.y;
      gi.ehi = r2.x;
    }
    const int32_t v = lane < gi.count ? __ldcg(f.list + gi.list_start + lane) : 0;
    expand_range<M>(a, h, gi.count, v, gi.elo, gi.ehi, s_T, s_B, lane, ws, acc);
  }

  // ---- phase 2b: dense small region (after a bitmap-mode level whose
  // frontier covers most small-degree vertices): the rows of the whole small
  // region are one contiguous col_idx range, cut at layout time into tasks
  // inside one degree class d; a warp streams a task with 128-bit loads and
  // keeps an element when its owner v = lo_d + (p - base_d) / d is in the
  // frontier bitmap. No list, no per-vertex row_ptr read.
  if (phases & 32) {
    for (int64_t it = gwarp; it < f.n_dense; it += nwarps) {
      const DenseTask dt = f.dense[it];
      const int d = dt.d;
      const int32_t lo = s_T[d + 1];
      const int64_t base = s_B[d];
      const uint32_t rcp = (uint32_t)(0xFFFFFFFFull / (uint32_t)d + 1ull);
      const int64_t a0 = dt.p0 & ~int64_t(3), a1 = dt.p0 + dt.len;
      for (int64_t c0 = a0; c0 < a1; c0 += 128) {
        const int64_t p = c0 + lane * 4;
        const int4 x = p < a1 ? ld_stream4(a.col_idx + p) : make_int4(0, 0, 0, 0);
        int32_t nb[4] = {x.x, x.y, x.z, x.w};
        int32_t own[4];
        uint32_t okm = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t pq = p + q;
          const uint32_t rel = (uint32_t)(pq - base);
          own[q] = lo + (d == 1 ? (int32_t)rel : (int32_t)__umulhi(rel, rcp));
          const bool in_task = pq >= dt.p0 && pq < a1;
          // (the frontier bitmap is read-only during a k_expand launch: through L1;
        // k_bfs rewrites it within its launch: through L2)
        const uint32_t fw = !in_task ? 0u : (f.front_nc ? __ldg(f.front + (own[q] >> 5)) : __ldcg(f.front + (own[q] >> 5)));
        const bool in_front = in_task && ((fw >> (own[q] & 31)) & 1u);
          okm |= (uint32_t)in_front << q;
          nb[q] = in_front ? nb[q] : 0;
        }
        probe_batch<M, 4>(a, h, nb, okm, [&](int k) { return __ldg(a.new2old + own[k]); }, lane, acc);
      }
    }
  }

  // ---- phase 2c: dense warp-bin region (32 <= deg < kCtaMin): a warp takes
  // 32 consecutive rows (contiguous in col_idx), skips the group when none of
  // them is in the frontier, else streams the group with 128-bit loads. The
  // owner of an element comes from a 128-bit mask of row starts in the
  // window (four redux.or) and a prefix popcount — no search, no list.
  if (phases & 64) {
    const int64_t ngroups = (a.t_warp - a.t_cta + 31) / 32;
    for (int64_t g = gwarp; g < ngroups; g += nwarps) {
      const int64_t v0 = a.t_cta + 32 * g;
      const int nrow = (int)std::min<int64_t>(32, a.t_warp - v0);
      // frontier bits of rows v0 .. v0+31 (two words when v0 is unaligned)
      const uint32_t sh = (uint32_t)(v0 & 31);
      const uint32_t wlo = __ldca(f.front + (v0 >> 5));
      const uint32_t whi = sh ? __ldca(f.front + (v0 >> 5) + 1) : 0u;
      uint32_t fw = sh ? ((wlo >> sh) | (whi << (32 - sh))) : wlo;
      fw &= (nrow == 32) ? kFull : ((1u << nrow) - 1u);
      if (!fw) continue;
      if (a.dbg && lane == 0) atomicAdd(a.dbg + 3, (unsigned long long)__popc(fw));  // LBFS_COUNT: frontier rows
      const int64_t rs = lane < nrow ? __ldg(a.row_ptr + v0 + lane) : 0;  // row starts
      const int64_t e_beg = __shfl_sync(kFull, rs, 0);
      const int64_t e_end = __ldg(a.row_ptr + v0 + nrow);  // (a 33rd lane does not exist)
      const int32_t uo = (lane < nrow && ((fw >> lane) & 1u)) ? __ldg(a.new2old + v0 + lane) : 0;
      for (int64_t c0 = e_beg & ~int64_t(3); c0 < e_end; c0 += 128) {
        const int64_t p = c0 + lane * 4;
        const int4 x = p < e_end ? ld_stream4(a.col_idx + p) : make_int4(0, 0, 0, 0);
        // row starts inside [c0, c0+128) as a 128-bit mask
        const int64_t off = rs - c0;
        const bool inwin = lane < nrow && off >= 0 && off < 128;
        uint32_t Mk[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          Mk[k] = __reduce_or_sync(kFull, (inwin && (off >> 5) == k) ? (1u << (off & 31)) : 0u);
        const int before = __popc(__ballot_sync(kFull, lane < nrow && off < 0));  // rows starting before c0
        const int wk = lane >> 3;  // this lane's 4 elements sit in mask word wk
        int pre = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) pre += (k < wk) ? __popc(Mk[k]) : 0;
        const uint32_t mw = wk == 0 ? Mk[0] : (wk == 1 ? Mk[1] : (wk == 2 ? Mk[2] : Mk[3]));
        int32_t nb[4] = {x.x, x.y, x.z, x.w};
        int own[4];
        uint32_t okm = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int o = lane * 4 + q;
          own[q] = before + pre + __popc(mw & ((2u << (o & 31)) - 1u)) - 1;  // row index within the group
          const bool ok = (p + q) >= e_beg && (p + q) < e_end && own[q] >= 0 && ((fw >> (own[q] & 31)) & 1u);
          okm |= (uint32_t)ok << q;
          nb[q] = ok ? nb[q] : 0;
          own[q] &= 31;
        }
        int32_t par[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) par[q] = __shfl_sync(kFull, uo, own[q]);
        if (a.dbg) atomicAdd(a.dbg + 2, (unsigned long long)__popc(okm));  // LBFS_COUNT: kept elements
        probe_batch<M, 4>(a, h, nb, okm, [&](int k) { return par[k]; }, lane, acc);
      }
    }
  }

  // ---- phase 3: raw warp/small queues (after a queue-mode level): a warp
  // takes one warp-bin vertex or 32 small-bin vertices ---------------------
  if (phases & 4) {
    // heavy levels: warp-bin rows streamed like slices (the next row's
    // descriptor and D windows in flight), then the small rows by 32
    const bool rows_streamed = false;  // (streamed rows: 334 vs 370 GTEPS on S24; kept off)
    if (rows_streamed) stream_queue_rows<M>(a, h, f.warp, f.n_warp, gwarp, nwarps, lane, acc);
    const int64_t n_warp = rows_streamed ? 0 : f.n_warp;
    const int64_t ng = n_warp + (f.n_small + 31) / 32;
    for (int64_t g = gwarp; g < ng; g += nwarps) {
      const bool wb = g < n_warp;
      const int64_t base = wb ? g : (g - n_warp) * 32;
      const int n = wb ? 1 : (int)std::min<int64_t>(32, f.n_small - base);
      const int32_t v = lane < n ? __ldcg((wb ? f.warp : f.small) + base + lane) : 0;
      LBFS_DCHECK(!(lane < n) || (v >= 0 && (int64_t)v < a.chk_n), "queue entry");
      expand_range<M>(a, h, n, v, 0, 1 << 30, s_T, s_B, lane, ws, acc);
    }
  }
}

// One launch per level and bin set (host-driven level loop).
// Queue-mode launches run 512 threads per CTA: their winner path (election,
// row reads, bin appends for a batch of 4) needs more than the 64 registers
// a 1024-thread CTA leaves, and a queue level is latency-bound anyway.
// (So do the bitmap-mode group items: their double-buffered windows plus the
// parent stores spill at 64 registers.)
template <int M, int kPhases>
constexpr int expand_threads() { return (M == kQueueOut || M == kBitmapOut) ? 512 : kExpandThreads; }

template <int M, int kPhases>
__global__ void __launch_bounds__(expand_threads<M, kPhases>(), 1) k_expand(LevelArgs a, Frontier f, int32_t hot_words) {
  extern __shared__ __align__(128) uint8_t s_dyn[];
  __shared__ ExpandSmem s;
  griddep_launch();
  expand_init(s, a);
  // (the shared-window base is made opaque: left alone, the compiler
  // rematerialises it — S2UR + three uniform ops — next to every shared OR)
  uint32_t hot_base = smem_u32(s_dyn);
  asm volatile("" : "+r"(hot_base));
  const Hot h{reinterpret_cast<uint32_t*>(s_dyn), hot_base, hot_words};
  uint4* h4 = reinterpret_cast<uint4*>(h.s);
  const int hw4 = hot_words >> 2;  // hot_words is a multiple of 4
  if constexpr (M == kHeavy) {
    for (int i = threadIdx.x; i < hw4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    griddep_wait();  // (the prologue above overlaps the previous kernel's tail)
  } else {
    griddep_wait();
    hot_load(s, h, a.visited);
  }
  Acc acc;
  expand_phases<M, kPhases>(a, f, s, h, acc);
  flush_acc<M>(a, acc);
  hot_drain(s);
  if constexpr (M == kHeavy) {  // this CTA's blind ORs -> its stage row
    uint4* row = reinterpret_cast<uint4*>(a.stage) + (size_t)blockIdx.x * (a.stage_words >> 2);
    for (int i = threadIdx.x; i < hw4; i += blockDim.x) {
      uint4 x = h4[i];
      if (!a.stage_first) {
        const uint4 y = __ldcg(row + i);
        x.x |= y.x, x.y |= y.y, x.z |= y.z, x.w |= y.w;
      }
      __stcg(row + i, x);
    }
  }
}

// Heavy levels: visited |= OR of the CTAs' stage rows over the hot prefix.
// grid (ceil(hw4 / 256), ceil(rows / kMergeRows)): a thread ORs kMergeRows
// rows of one 16-byte column and folds the result in with red.or.
constexpr int kMergeRows = 16;
__global__ void __launch_bounds__(256) k_merge_hot(const uint4* __restrict__ stage, int rows, int hw4, int stride4,
                                                   uint32_t* __restrict__ visited) {
  griddep_launch();
  griddep_wait();
  const int i = blockIdx.x * 256 + threadIdx.x;
  if (i >= hw4) return;
  const int r0 = blockIdx.y * kMergeRows, r1 = min(rows, r0 + kMergeRows);
  uint4 x = make_uint4(0, 0, 0, 0);
#pragma unroll 8
  for (int r = r0; r < r1; ++r) {
    const uint4 y = __ldcg(stage + (size_t)r * stride4 + i);
    x.x |= y.x, x.y |= y.y, x.z |= y.z, x.w |= y.w;
  }
  uint32_t* w = visited + 4 * (size_t)i;
  if (x.x) red_or(w + 0, x.x);
  if (x.y) red_or(w + 1, x.y);
  if (x.z) red_or(w + 2, x.z);
  if (x.w) red_or(w + 3, x.w);
}

// ---------------------------------------------------------------- K3 compaction
// A block owns kCompactVerts consecutive internal ids (kCompactWords visited
// words): new = visited & ~prev. Hubs become kChunk slices; the other new
// vertices get list ranks in ascending id (prefix of per-word popcounts), so
// the list is id-ordered within the block and degree classes stay together;
// every 32 consecutive list entries form a group cut into kItemElems-element
// items. One atomic per output per block reserves space. Pass 2 (one vertex
// per thread per step, so new2old/row_ptr/pred_int reads coalesce) writes
// levels and parents in original ids and folds the K6 stats.
#ifndef LBFS_COMPACT_MINB
#define LBFS_COMPACT_MINB 1
#endif
constexpr int kCompactThreads = 256;
// ids per compaction block: 4096, or 2048 for small graphs (n < 4 M: the
// compaction of a small graph is a handful of blocks per SM, each a chain of
// scans and barriers — smaller blocks shorten the chain: S20 +3%; S24 -3%)
constexpr int kCompactVertsBig = 4096, kCompactVertsSmall = 2048;
constexpr int64_t kCompactSmallGraph = (int64_t)1 << 22;
constexpr int kCompactSparseDiv = 8;  // pass 2 walks only the new ids when fewer than 1/8 of the block's ids are new

// A compaction group is 256 threads synchronised on named barrier `bar`
// (a whole CTA in k_compact; a quarter of a k_bfs CTA).
__device__ __forceinline__ void gsync(int bar) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(kCompactThreads) : "memory");
}
__device__ __forceinline__ int gsync_or(int bar, bool pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 p, %2, 0;\n\t"
      "bar.red.or.pred q, %1, %3, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(bar), "r"((int)pred), "r"(kCompactThreads)
      : "memory");
  return r;
}

// exclusive scan of one int per thread over the first 128 threads of the
// group (all 256 must call); returns the exclusive prefix, *total the sum
__device__ __forceinline__ int scan128(int t, int bar, int val, int* s_w, int* total) {
  const int lane = t & 31;
  int incl = val;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += x;
  }
  gsync(bar);
  if (t < 128 && lane == 31) s_w[t >> 5] = incl;
  gsync(bar);
  int before = 0;
  for (int k = 0; k < (t >> 5) && k < 4; ++k) before += s_w[k];
  *total = s_w[0] + s_w[1] + s_w[2] + s_w[3];
  return before + incl - val;
}

template <int V>
struct CompactSmem {
  unsigned long long base[4];
  unsigned long long red[3][kCompactThreads / 32];
  uint32_t new_[V / 32];
  uint32_t lmask[V / 32];
  int32_t lpre[V / 32];
  int32_t npre[V / 32];  // exclusive prefix of new vertices per word
  uint32_t wmask[V / 32];
  int32_t wpre[V / 32];
  int32_t gsum[V / 32];
  int32_t hitems[V / 32];  // hub slices per word, then their word offsets
  int32_t w[4];
  int32_t deg[V];
};

// One compaction block (kCompactVerts ids) by a 256-thread group: thread t
// of the group, named barrier `bar`, shared scratch sm.
template <int V>
__device__ __forceinline__ void compact_block(const CompactArgs& c, int64_t blk, CompactSmem<V>& sm, int t, int bar) {
  constexpr int kCompactVerts = V, kCompactWords = V / 32, kCompactSteps = V / kCompactThreads;
  uint32_t* s_new = sm.new_;
  uint32_t* s_lmask = sm.lmask;
  int32_t* s_lpre = sm.lpre;
  uint32_t* s_wmask = sm.wmask;
  int32_t* s_wpre = sm.wpre;
  int32_t* s_deg = sm.deg;
  int32_t* s_gsum = sm.gsum;
  int32_t* s_w = sm.w;
  unsigned long long* s_base = sm.base;
  int32_t* s_hitems = sm.hitems;
  const int lane = t & 31, warp = t >> 5;
  const int64_t w0 = blk * kCompactWords;
  const int64_t v0 = w0 * 32;
  gsync(bar);  // the previous block's readers of sm are done
  uint32_t nb = 0, mhub = 0, mlist = 0, mwarp = 0;
  if (t < kCompactWords) s_hitems[t] = 0;
  if (t < kCompactWords && w0 + t < c.nwords) {
    const int64_t gw = ((w0 + t) << c.part_log) | c.part_rank;  // global word of owned word w0+t
    const uint32_t w = __ldcg(c.visited + gw), p = __ldcg(c.prev + gw);
    nb = w & ~p;
    c.front[w0 + t] = nb;  // next frontier as a bitmap (dense small-region path)
    if (c.fsend) c.fsend[w0 + t] = nb;
    if (nb) {
      c.prev[gw] = w;
      const int64_t vw = (w0 + t) * 32;
      mhub = nb & range_mask(vw, 0, c.t_cta);
      mwarp = nb & range_mask(vw, c.t_cta, c.t_warp);
      mlist = nb & range_mask(vw, c.t_warp, c.t_nz);
    }
  }
  const int any_hub = gsync_or(bar, mhub != 0);  // (also orders s_hitems' zeroing)
  if (!gsync_or(bar, nb != 0)) return;
  if (t < kCompactWords) {
    s_new[t] = nb;
    s_lmask[t] = mlist;
    s_wmask[t] = mwarp;
  }
  // one scan for the list and warp-slice ranks (packed 16 | 16: a block has
  // <= 4096 ids), one for the rank of every new vertex (pass 2 walks only those)
  int n_list = 0, n_wsl = 0, n_new = 0, packed_tot = 0;
  const int ppre = scan128(t, bar, __popc(mlist) | (__popc(mwarp) << 16), s_w, &packed_tot);
  n_list = packed_tot & 0xFFFF;
  n_wsl = packed_tot >> 16;
  if (t < kCompactWords) {
    s_lpre[t] = ppre & 0xFFFF;
    s_wpre[t] = ppre >> 16;
  }
  const int npre = scan128(t, bar, __popc(nb), s_w, &n_new);
  if (t < kCompactWords) sm.npre[t] = npre;
  if (t == 0) {
    s_base[0] = n_list ? atomicAdd(&c.next_cnt->bin[kBinSmall], (unsigned long long)n_list) : 0;
    s_base[3] = n_wsl ? atomicAdd(&c.next_cnt->bin[kBinWSlice], (unsigned long long)n_wsl) : 0;
  }
  gsync(bar);
  // pass 2. Dense blocks (most ids new): thread t owns vertices v0 + t + 256 j
  // (bit t&31 of word t/32 + 8 j). Sparse blocks: the block's new vertices in
  // ascending order, new vertex i to thread i % 256 (word by binary search over
  // the new-vertex ranks, bit by select), so no step waits on loads for ids
  // that are not new. Four vertices' loads are issued before any of their stores.
  unsigned long long edges = 0, big = 0;
  auto settle_new = [&](int wl, int b, int64_t st, int64_t en, int32_t vo) {
    const int64_t v = v0 + wl * 32 + b;
    c.level_int[v] = c.next_level;  // outputs are written by k_finalize
    const int32_t deg = (int32_t)(en - st);
    edges += (unsigned long long)deg;
    if (v < c.t_warp) big += (unsigned long long)deg;
    const uint32_t wm = s_wmask[wl];
    if ((wm >> b) & 1u)  // warp-bin row: one slice, parent = the row's vertex
      c.next_wslice[s_base[3] + s_wpre[wl] + __popc(wm & ((1u << b) - 1u))] = CtaItem{st, deg, vo};
    const uint32_t lm = s_lmask[wl];
    if ((lm >> b) & 1u) {
      const int r = s_lpre[wl] + __popc(lm & ((1u << b) - 1u));
      c.next_list[s_base[0] + r] = (int32_t)v;
      s_deg[r] = deg;
    }
    if (v < c.t_cta) atomicAdd(&s_hitems[wl], slice_items(st, deg, kChunk));
  };
  if (n_new * kCompactSparseDiv > kCompactVerts) {
#pragma unroll 1
    for (int j0 = 0; j0 < kCompactSteps; j0 += 4) {
      int64_t st[4], en[4];
      int32_t vo[4];
      bool nw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int wl = (t >> 5) + (j0 + q) * (kCompactThreads / 32);
        const int64_t v = v0 + t + (j0 + q) * kCompactThreads;
        nw[q] = (s_new[wl] >> (t & 31)) & 1u;
        vo[q] = nw[q] && v >= c.t_cta && v < c.t_warp ? __ldg(c.new2old + v) : 0;
        st[q] = nw[q] ? __ldg(c.row_ptr + v) : 0;
        en[q] = nw[q] ? __ldg(c.row_ptr + v + 1) : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (nw[q]) settle_new((t >> 5) + (j0 + q) * (kCompactThreads / 32), t & 31, st[q], en[q], vo[q]);
    }
  } else {
#pragma unroll 1
    for (int i0 = 0; i0 < n_new; i0 += 4 * kCompactThreads) {
      int64_t st[4], en[4];
      int32_t vo[4];
      int wlq[4], bq[4];
      bool nw[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = i0 + q * kCompactThreads + t;
        nw[q] = i < n_new;
        int wl = 0;
#pragma unroll
        for (int step = kCompactWords / 2; step; step >>= 1)  // largest wl with npre[wl] <= i
          if (sm.npre[wl + step] <= i) wl += step;
        uint32_t m = s_new[wl];
        int k = i - sm.npre[wl], pos = 0;
#pragma unroll
        for (int half = 16; half; half >>= 1) {  // position of the k-th set bit of m
          const int cnt = __popc(m & ((1u << half) - 1u));
          const bool up = k >= cnt;
          k -= up ? cnt : 0;
          m = up ? m >> half : m;
          pos += up ? half : 0;
        }
        wlq[q] = wl;
        bq[q] = pos;
        const int64_t v = v0 + wl * 32 + pos;
        vo[q] = nw[q] && v >= c.t_cta && v < c.t_warp ? __ldg(c.new2old + v) : 0;
        st[q] = nw[q] ? __ldg(c.row_ptr + v) : 0;
        en[q] = nw[q] ? __ldg(c.row_ptr + v + 1) : 0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (nw[q]) settle_new(wlq[q], bq[q], st[q], en[q], vo[q]);
    }
  }
  const int b = t & 31;
  if (c.resolve_verts > v0) {
    // heavy level: the new hot vertices were discovered by blind ORs with no
    // parent; take the first neighbour one level up (rows are sorted by
    // internal id, i.e. by descending degree: the first entry is usually it).
    // Any such neighbour is a valid parent (traversal.py:145-147).
#pragma unroll 1
    for (int j0 = 0; j0 < kCompactSteps; j0 += 8) {
      int32_t u[8], lv[8];
      bool need[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {  // first neighbour (precomputed per row: coalesced)
        const int wl = (t >> 5) + (j0 + q) * (kCompactThreads / 32);
        const int64_t v = v0 + t + (j0 + q) * kCompactThreads;
        need[q] = v < c.resolve_verts && ((s_new[wl] >> b) & 1u);
        u[q] = need[q] ? __ldg(c.first_nbr + v) : 0;
      }
#pragma unroll
      // through L1: most first neighbours are a few hubs (an L2 hot spot otherwise);
      // frontier entries (level cur_level) were written by an earlier launch, and a
      // stale copy of an entry written now reads -1, never cur_level
      for (int q = 0; q < 8; ++q) lv[q] = need[q] ? __ldg(c.level_int + u[q]) : -1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        if (!need[q]) continue;
        const int64_t v = v0 + t + (j0 + q) * kCompactThreads;
        int32_t par = kSentinel;
        if (lv[q] == c.cur_level) {
          par = __ldg(c.new2old + u[q]);
        } else {  // rare: scan the rest of the row
          const int64_t p = __ldg(c.row_ptr + v), e = __ldg(c.row_ptr + v + 1);
          for (int64_t k = p + 1; k < e; ++k) {
            const int32_t x = __ldg(c.col_idx + k);
            if (__ldg(c.level_int + x) == c.cur_level) {
              par = __ldg(c.new2old + x);
              break;
            }
          }
        }
        c.pred_int[v] = par;
      }
    }
  }
  gsync(bar);
  if (any_hub) {
    // hub slices: word offsets from one scan, slots inside a word claimed
    // with shared atomics (slice order is free); one vertex per thread per
    // step, so the row_ptr reads stay parallel (they hit L1: read above)
    int n_hub_items = 0;
    const int hi = t < kCompactWords ? s_hitems[t] : 0;
    const int ipre = scan128(t, bar, hi, s_w, &n_hub_items);
    gsync(bar);
    if (t < kCompactWords) s_hitems[t] = ipre;
    if (t == 0) s_base[1] = atomicAdd(&c.next_cnt->bin[kBinCta], (unsigned long long)n_hub_items);
    gsync(bar);
    for (int j = 0; j < kCompactSteps; ++j) {
      const int wl = (t >> 5) + j * (kCompactThreads / 32);
      const int64_t v = v0 + t + j * kCompactThreads;
      if (v >= c.t_cta || !((s_new[wl] >> b) & 1u)) continue;
      const int64_t st = __ldg(c.row_ptr + v), deg = __ldg(c.row_ptr + v + 1) - st;
      const int items = slice_items(st, (int32_t)deg, kChunk);
      const int32_t vo = __ldg(c.new2old + v);
      unsigned long long p = s_base[1] + atomicAdd(&s_hitems[wl], items);
      for (int k = 0; k < items; ++k) c.next_cta[p++] = slice_item(st, (int32_t)deg, kChunk, k, vo);
    }
  }
  // groups of 32 consecutive list entries -> kItemElems-element items
  const int ngroups = (n_list + 31) / 32;
  for (int g = warp; g < ngroups; g += kCompactThreads / 32) {
    const int r = g * 32 + lane;
    int x = r < n_list ? s_deg[r] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(kFull, x, o);
    if (lane == 0) s_gsum[g] = x;
  }
  gsync(bar);
  const int gsum = t < ngroups ? s_gsum[t] : 0;
  const int nsub = t < ngroups ? std::max(1, (gsum + kItemElems - 1) / kItemElems) : 0;
  int n_items = 0;
  const int gpre = scan128(t, bar, nsub, s_w, &n_items);
  if (t == 0) s_base[2] = atomicAdd(&c.next_cnt->bin[kBinItems], (unsigned long long)n_items);
  gsync(bar);
  for (int k = 0; k < nsub; ++k) {
    GroupItem gi;
    gi.list_start = (int64_t)s_base[0] + 32 * t;
    gi.count = std::min(32, n_list - 32 * t);
    gi.elo = k * kItemElems;
    gi.ehi = std::min(gsum, (k + 1) * kItemElems);
    gi.pad = 0;
    c.next_items[s_base[2] + gpre + k] = gi;
  }
  unsigned long long e = edges, d = (unsigned long long)__popc(nb), bg = big;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    e += __shfl_xor_sync(kFull, e, o);
    d += __shfl_xor_sync(kFull, d, o);
    bg += __shfl_xor_sync(kFull, bg, o);
  }
  if (lane == 0) {
    sm.red[0][warp] = e;
    sm.red[1][warp] = d;
    sm.red[2][warp] = bg;
  }
  gsync(bar);
  if (t == 0) {
    unsigned long long e_tot = 0, d_tot = 0, b_tot = 0;
    for (int k = 0; k < kCompactThreads / 32; ++k) {
      e_tot += sm.red[0][k];
      d_tot += sm.red[1][k];
      b_tot += sm.red[2][k];
    }
    if (e_tot) atomicAdd(&c.next_cnt->edges, e_tot);
    if (d_tot) atomicAdd(&c.next_cnt->discovered, d_tot);
    if (b_tot) atomicAdd(&c.next_cnt->big_edges, b_tot);
  }
}

template <int V>
__global__ void __launch_bounds__(kCompactThreads, LBFS_COMPACT_MINB) k_compact(CompactArgs c) {
  griddep_launch();
  griddep_wait();
  __shared__ CompactSmem<V> sm;
  compact_block<V>(c, blockIdx.x, sm, threadIdx.x, 1);
}



// ---------------------------------------------------------------- K4 init
// per-BFS state: visited/prev bitmaps cleared, internal levels -1
__device__ __forceinline__ void init_range(uint4* __restrict__ vis4, uint4* __restrict__ prev4, int64_t nwords4,
                                           int4* __restrict__ lvl4, int64_t n4, int64_t t, int64_t stride) {
  for (int64_t i = t; i < nwords4; i += stride) vis4[i] = prev4[i] = make_uint4(0, 0, 0, 0);
  const int4 m4 = make_int4(-1, -1, -1, -1);
  for (int64_t i = t; i < n4; i += stride) lvl4[i] = m4;
}
__global__ void k_init(uint4* __restrict__ vis4, uint4* __restrict__ prev4, int64_t nwords4,
                       int4* __restrict__ lvl4, int64_t n4, Counters* __restrict__ ring) {
  init_range(vis4, prev4, nwords4, lvl4, n4, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
             (int64_t)gridDim.x * blockDim.x);
  // (host-driven BFS) the counter ring cleared here instead of by a memset
  if (ring && blockIdx.x == 0 && threadIdx.x < (int)(kCounterRing * sizeof(Counters) / 8))
    reinterpret_cast<unsigned long long*>(ring)[threadIdx.x] = 0ull;
}

// K4 for one unpartitioned BFS in one launch: k_init with the root seeded in
// place (its visited / prev bit and level 0 are written by the threads that
// clear those words), the rest of seed_root by thread 0 of block 0 after the
// ring is cleared. Saves the one-thread k_seed launch.
__global__ void k_init_seed(uint4* __restrict__ vis4, uint4* __restrict__ prev4, int64_t nwords4,
                            int4* __restrict__ lvl4, int64_t n4, Counters* __restrict__ ring, LevelArgs a,
                            const int32_t* __restrict__ old2new, int32_t root_orig) {
  griddep_launch();
  const int32_t r = __ldg(old2new + root_orig);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t rw4 = (int64_t)(r >> 5) >> 2, rl4 = (int64_t)r >> 2;
  for (int64_t i = t; i < nwords4; i += stride) {
    const uint32_t bit = i == rw4 ? 1u << (r & 31) : 0u;
    const int sel = (r >> 5) & 3;
    vis4[i] = prev4[i] = make_uint4(sel == 0 ? bit : 0u, sel == 1 ? bit : 0u, sel == 2 ? bit : 0u, sel == 3 ? bit : 0u);
  }
  for (int64_t i = t; i < n4; i += stride) {
    const int hit = i == rl4 ? (r & 3) : -1;
    lvl4[i] = make_int4(hit == 0 ? 0 : -1, hit == 1 ? 0 : -1, hit == 2 ? 0 : -1, hit == 3 ? 0 : -1);
  }
  if (blockIdx.x != 0) return;
  if (threadIdx.x < (int)(kCounterRing * sizeof(Counters) / 8))
    reinterpret_cast<unsigned long long*>(ring)[threadIdx.x] = 0ull;
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t st = a.row_ptr[r];
    const int32_t deg = (int32_t)(a.row_ptr[r + 1] - st);
    a.pred_int[r] = root_orig;
    Counters c{};
    c.discovered = 1;
    c.edges = (unsigned long long)deg;
    if (r < a.t_cta) {
      const int items = slice_items(st, deg, a.qchunk);
      for (int k = 0; k < items; ++k) a.next_cta[k] = slice_item(st, deg, a.qchunk, k, root_orig);
      c.bin[kBinCta] = (unsigned long long)items;
    } else if (r < a.t_warp) {
      a.next_warp[0] = r;
      c.bin[kBinWarp] = 1;
    } else if (r < a.t_nz) {
      a.next_small[0] = r;
      c.bin[kBinSmall] = 1;
    }
    ring[0] = c;
  }
}

// Outputs in original ids, once per BFS (PredecessorArray semantics,
// traversal.py:42-50: unreached and padding = SENTINEL): output x takes the
// record of internal id old2new[x]; reached = its visited bit (a 2 MiB
// bitmap that stays in L2), so only reached vertices read their parent.
// Sequential 128-bit writes over [x0, x1) (x0 % 4 == 0); kVec: 16-byte
// aligned output (else scalar stores).
template <bool kVec>
__global__ void __launch_bounds__(256) k_finalize(const int32_t* __restrict__ old2new, const uint32_t* __restrict__ visited,
                                                  const int32_t* __restrict__ rec, int32_t miss, int64_t n, int64_t x0,
                                                  int64_t x1, int32_t* __restrict__ out) {
  const int64_t i0 = x0 / 4, i1 = (x1 + 3) / 4;
  for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < i1; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v4 = __ldg(reinterpret_cast<const int4*>(old2new) + i);  // (old2new is padded to 4)
    const int32_t v[4] = {v4.x, v4.y, v4.z, v4.w};
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = i * 4 + q < n ? __ldg(visited + (v[q] >> 5)) : 0u;
    int32_t r[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) r[q] = ((w[q] >> (v[q] & 31)) & 1u) ? __ldg(rec + v[q]) : miss;
    if (kVec && i * 4 + 3 < x1) {
      reinterpret_cast<int4*>(out)[i] = make_int4(r[0], r[1], r[2], r[3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i * 4 + q >= x0 && i * 4 + q < x1) out[i * 4 + q] = r[q];
    }
  }
}

// Root of a BFS (traversal.py:135-139, 343-347): its bit in visited/prev
// (and in the replicated frontier bitmap when partitioned) on every rank;
// the owner records level 0 / pred = root and seeds its bins. red, when
// given, receives the (frontier, edges) counts for the cross-rank sum.
__device__ __forceinline__ void seed_root(const LevelArgs& a, uint32_t* prev, const int32_t* old2new,
                                          int32_t root_orig, Counters* cnt0, uint32_t* fglob,
                                          unsigned long long* red) {
  const int32_t r = old2new[root_orig];
  a.visited[r >> 5] |= 1u << (r & 31);
  prev[r >> 5] |= 1u << (r & 31);
  if (fglob) fglob[r >> 5] |= 1u << (r & 31);
  Counters c{};
  if (part_owned(r, a.part_log, a.part_rank)) {
    const int32_t l = part_local(r, a.part_log);
    const int64_t st = a.row_ptr[l];
    const int32_t deg = (int32_t)(a.row_ptr[l + 1] - st);
    a.level_int[l] = 0;
    a.pred_int[l] = root_orig;
    c.discovered = 1;
    c.edges = (unsigned long long)deg;
    if (l < a.t_cta) {
      const int items = slice_items(st, deg, a.qchunk);
      for (int k = 0; k < items; ++k) a.next_cta[k] = slice_item(st, deg, a.qchunk, k, root_orig);
      c.bin[kBinCta] = (unsigned long long)items;
    } else if (l < a.t_warp) {
      a.next_warp[0] = l;
      c.bin[kBinWarp] = 1;
    } else if (l < a.t_nz) {
      a.next_small[0] = l;
      c.bin[kBinSmall] = 1;
    }
  }
  *cnt0 = c;
  if (red) {
    red[0] = c.discovered;
    red[1] = c.edges;
  }
}
__global__ void k_seed(LevelArgs a, uint32_t* prev, const int32_t* old2new, int32_t root_orig, Counters* cnt0,
                       uint32_t* fglob, unsigned long long* red) {
  seed_root(a, prev, old2new, root_orig, cnt0, fglob, red);
}

// End of a host-driven level: the next frontier's counters go to the host
// mailbox (mapped pinned memory) behind a sequence number, and the ring slot
// the following level writes is cleared.
__global__ void k_publish(Counters* ring, int slot, int zero_slot, Counters* mail, unsigned long long* seq,
                          unsigned long long value) {
  const int t = threadIdx.x;
  constexpr int kWords = (int)(sizeof(Counters) / 8);
  griddep_wait();
  if (t < kWords) {
    reinterpret_cast<volatile unsigned long long*>(mail)[t] = reinterpret_cast<unsigned long long*>(&ring[slot])[t];
    reinterpret_cast<unsigned long long*>(&ring[zero_slot])[t] = 0ull;
  }
  __syncwarp();
  if (t == 0) {
    __threadfence_system();
    *reinterpret_cast<volatile unsigned long long*>(seq) = value;
  }
}

void BfsEngine::publish_and_wait(int slot, int zero_slot, cudaStream_t st) {
  const unsigned long long want = ++seq_;
  LBFS_LAUNCH_PDL(k_publish, 1, 32, 0, st, cnt_, slot, zero_slot, h_mail_, h_seq_, want);
  flush_resolve(st);
  wait_mail(want, st);
  std::atomic_thread_fence(std::memory_order_acquire);  // (the counters are read after the sequence word)
  h_cnt_[slot] = *const_cast<const Counters*>(h_mail_);
}

void BfsEngine::wait_mail(unsigned long long want, cudaStream_t st) {
  // spin: a blocking stream sync costs tens of microseconds of wake-up per level
  volatile unsigned long long* p = h_seq_;
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spins = 1; *p < want; ++spins) {
    if ((spins & 0x3FFF) == 0) {
      const cudaError_t e = cudaStreamQuery(st);
      if (e != cudaSuccess && e != cudaErrorNotReady) throw_cuda(e, "level kernels", __FILE__, __LINE__);
      if (e == cudaSuccess && *p < want) throw Failure(LBFS_ECUDA, "internal: level mailbox not written");
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        throw Failure(LBFS_ECUDA, "level did not complete within 120 s");
    }
  }
}

// ---------------------------------------------------------------- engine
BfsEngine::BfsEngine(const Csr& csr, int rank, int nparts) {
  if (nparts < 1 || (nparts & (nparts - 1)) != 0 || nparts > 64) throw_inval("nparts must be a power of two <= 64");
  if (rank < 0 || rank >= nparts) throw_inval("rank out of range");
  LBFS_CUDA(cudaGetDevice(&device_));
  sm_count_ = current_sm_count();
  nparts_ = nparts;
  part_rank_ = rank;
  while ((1 << part_log_) < nparts_) ++part_log_;
  n_ = csr.n;
  nnz_ = csr.nnz;
  // bitmap words rounded up to whole partition rounds; rank g owns words g, g+P, ...
  nwords_ = ((n_ + 31) / 32 + nparts_ - 1) / nparts_ * nparts_;
  nwl_ = nwords_ / nparts_;
  n_loc_ = nparts_ == 1 ? n_ : nwl_ * 32;
  npad_ = pad32(n_);
  {
    // (experiment, off: level kernels at the highest stream priority and the
    // side work at the lowest measured 385 vs 389 GTEPS at equal priorities)
    int prio_lo = 0, prio_hi = 0;
    LBFS_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    const bool prio = env_flag("LBFS_STREAM_PRIO");
    LBFS_CUDA(cudaStreamCreateWithPriority(&stream_, cudaStreamNonBlocking, prio ? prio_hi : 0));
    LBFS_CUDA(cudaStreamCreateWithPriority(&res_st_, cudaStreamNonBlocking, prio ? prio_lo : 0));
  }
  LBFS_CUDA(cudaEventCreateWithFlags(&ev_resolve_, cudaEventDisableTiming));
  LBFS_CUDA(cudaEventCreateWithFlags(&ev_side_done_, cudaEventDisableTiming));
  for (auto& e : ev_snap_) LBFS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  build_layout(csr);
  visited_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
  prev_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
  pred_int_ = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_loc_, 1));
  level_int_ = dev_alloc<int32_t>((size_t)(n_loc_ + 4));
  front_ = dev_alloc<uint32_t>((size_t)nwl_ + 4);
  dbg_ = dev_alloc<unsigned long long>(4);
  LBFS_CUDA(cudaMemset(dbg_, 0, 4 * sizeof(unsigned long long)));
  if (nparts_ > 1) {
    fglob_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
    resolve_cnt_ = dev_alloc<unsigned long long>(1);
    LBFS_CUDA(cudaMemset(resolve_cnt_, 0, sizeof(unsigned long long)));
  }
  // Bins, double-buffered: a vertex enters a bin once per BFS, so n entries
  // bound the small/warp bins; CTA items <= nnz/kChunk + #(deg >= kCtaMin).
  // (queue-mode winners also emit warp-bin rows as items; aligned cuts add at most one item per row)
  cap_cta_ = nnz_loc_ / kQChunkMin + 2 * (int64_t)t_warp_ + 2;
  // group items: one per started kItemElems of each 32-entry group, per block
  cap_items_ = nnz_loc_ / kItemElems + n_loc_ / 32 + 2 * ((n_loc_ + kCompactVertsSmall - 1) / kCompactVertsSmall) + 16;
  for (int b = 0; b < 2; ++b) {
    q_small_[b] = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_loc_, 1));
    q_warp_[b] = dev_alloc<int32_t>((size_t)std::max<int64_t>(t_warp_, 1));
    q_cta_[b] = dev_alloc<CtaItem>((size_t)cap_cta_);
    q_items_[b] = dev_alloc<GroupItem>((size_t)cap_items_);
    q_wslice_[b] = dev_alloc<CtaItem>((size_t)std::max<int64_t>(t_warp_ - t_cta_, 1));
  }
  cnt_ = dev_alloc<Counters>(kCounterRing);
  LBFS_CUDA(cudaMallocHost(&h_cnt_, sizeof(Counters) * kCounterRing));
  {
    void* m = nullptr;
    LBFS_CUDA(cudaHostAlloc(&m, sizeof(Counters) + 64, cudaHostAllocMapped));
    memset(m, 0, sizeof(Counters) + 64);
    h_mail_ = reinterpret_cast<Counters*>(m);
    h_seq_ = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(m) + sizeof(Counters));
  }
  for (auto& e : ev_) LBFS_CUDA(cudaEventCreate(&e));
  for (auto& e : ev_split_) LBFS_CUDA(cudaEventCreate(&e));
  LBFS_CUDA(cudaEventCreate(&ev_gap_));
  for (auto& e : ev_cl_) LBFS_CUDA(cudaEventCreate(&e));
  int occ = 0;
  // shared memory: the TMA ring plus as much of the visited bitmap as fits
  // (static shared memory differs per phase kernel: take the largest)
  const void* kernels[] = {(const void*)k_expand<kBitmapOut, 1>,  (const void*)k_expand<kBitmapOut, 2>,
                           (const void*)k_expand<kBitmapOut, 4>,
                           (const void*)k_expand<kBitmapOut, 16>, (const void*)k_expand<kBitmapOut, 32>,
                           (const void*)k_expand<kBitmapOut, 64>, (const void*)k_expand<kQueueOut, 1>,
                           (const void*)k_expand<kQueueOut, 2>,   (const void*)k_expand<kQueueOut, 4>,
                           (const void*)k_expand<kQueueOut, 16>,
                           (const void*)k_expand<kQueueOut, 32>,  (const void*)k_expand<kQueueOut, 64>,
                           (const void*)k_expand<kHeavy, 1>,      (const void*)k_expand<kHeavy, 2>,
                           (const void*)k_expand<kHeavy, 4>,
                           (const void*)k_expand<kHeavy, 16>,     (const void*)k_expand<kHeavy, 32>,
                           (const void*)k_expand<kHeavy, 64>,     (const void*)k_expand<kHeavy, 5>,
                           (const void*)k_expand<kQueueOut, 5>};
  size_t max_static = 0;
  for (auto fn : kernels) {
    cudaFuncAttributes fa{};
    LBFS_CUDA(cudaFuncGetAttributes(&fa, fn));
    max_static = std::max(max_static, fa.sharedSizeBytes);
  }
  int optin = 0;
  LBFS_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device_));
  int64_t avail = (int64_t)optin - (int64_t)max_static - 1024;
  {  // the sweep kernel's ring + static part must fit next to the same hot prefix
    cudaFuncAttributes fs{};
    LBFS_CUDA(cudaFuncGetAttributes(&fs, (const void*)k_sweep));
    avail = std::min<int64_t>(avail, (int64_t)optin - (int64_t)fs.sharedSizeBytes - kSweepRingBytes);
  }
  hot_words_ = (int32_t)std::min<int64_t>(std::max<int64_t>(avail / 4, 0) & ~int64_t(3), (nwords_ + 3) & ~int64_t(3));
  dyn_smem_ = hot_words_ * 4;
  for (auto fn : kernels) LBFS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem_));
  LBFS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_expand<kBitmapOut, 2>, kExpandThreads, dyn_smem_));
  expand_grid_ = sm_count_ * std::max(occ, 1);
  if (hot_words_ >= 4) {
    // the sweep has no per-warp rings: its hot prefix takes what its own ring leaves
    cudaFuncAttributes fs{};
    LBFS_CUDA(cudaFuncGetAttributes(&fs, (const void*)k_sweep));
    const int64_t sw_avail = (int64_t)optin - (int64_t)fs.sharedSizeBytes - kSweepRingBytes;
    sweep_hot_words_ = (int32_t)std::max<int64_t>(
        hot_words_, std::min<int64_t>((sw_avail / 4) & ~int64_t(3), (nwords_ + 3) & ~int64_t(3)));
    // the window stream keeps nothing but the hot prefix in shared memory
    stream_hot_words_ = (int32_t)std::min<int64_t>((((int64_t)optin - 1024) / 4) & ~int64_t(3),
                                                   (nwords_ + 3) & ~int64_t(3));
    stage_words_ = std::max(sweep_hot_words_, stream_hot_words_);
    stage_ = dev_alloc<uint32_t>((size_t)expand_grid_ * stage_words_);
    LBFS_CUDA(cudaFuncSetAttribute((const void*)k_stream_heavy<kStreamDepth>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, stream_hot_words_ * 4));
    if (n_side_win_ > 0) wmask_ = dev_alloc<uint4>((size_t)n_side_win_);
    sweep_fits_ = (int64_t)fs.sharedSizeBytes + kSweepRingBytes + (int64_t)sweep_hot_words_ * 4 <= optin;
    if (sweep_fits_)
      LBFS_CUDA(cudaFuncSetAttribute((const void*)k_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     kSweepRingBytes + sweep_hot_words_ * 4));
  }
  LBFS_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&h_loop_layers_), sizeof(lbfs_layer) * kLoopCap,
                          cudaHostAllocMapped));
  read_env();
  if (nparts_ == 1) setup_cluster(optin);
}

// Small-frontier levels: one cluster of cl_size_ CTAs (16 when the device
// allows non-portable cluster sizes, else 8), the visited bitmap dealt out to
// their shared memory when it fits next to the frontier queues.
void BfsEngine::setup_cluster(int optin) {
  const int64_t stat = (int64_t)cluster_static_smem();
  for (int cs : {cl_force_size_ ? cl_force_size_ : 16, 8}) {
    const int64_t nsec = (nwords_ + 7) / 8;
    const int64_t slice = (nsec + cs - 1) / cs * 8;  // words per CTA
    const int64_t budget = (int64_t)optin - stat - 1024 - (int64_t)kMaxCluster * kClusterStage * (int64_t)sizeof(QEntry);
    const int64_t qbytes = 2 * (int64_t)sizeof(QEntry);  // per queue slot (two queues)
    bool dsm = !cl_no_dsm_ && slice * 4 + qbytes * 1024 <= budget;
    // candidate mailboxes (DSMEM mode): mail_cap entries per sender, as many as
    // fit next to the slice and queues of >= 2048 entries (else remote claims)
    int64_t mail_cap = 0;
    if (dsm && !cl_no_mail_)
      for (int64_t c : {512, 256, 128})
        if (slice * 4 + (int64_t)kMaxCluster * c * 8 + qbytes * 2048 <= budget) {
          mail_cap = c;
          break;
        }
    if (mail_cap > 0 && cl_mail_cap_env_ > 0)  // (tests) a tiny region exercises the overflow path
      mail_cap = std::min<int64_t>(mail_cap, cl_mail_cap_env_);
    const int64_t mail_bytes = (int64_t)kMaxCluster * mail_cap * 8;
    int64_t qs = dsm ? std::min<int64_t>(8192, (budget - slice * 4 - mail_bytes) / qbytes)
                     : std::min<int64_t>(8192, budget / qbytes);
    qs &= ~int64_t(3);
    const void* fn = dsm ? (const void*)k_cluster_levels<true> : (const void*)k_cluster_levels<false>;
    const int smem = (int)((dsm ? slice * 4 : 0) + qbytes * qs + (int64_t)kMaxCluster * kClusterStage * sizeof(QEntry) +
                           mail_bytes);
    if (cs > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      (void)cudaGetLastError();
      continue;
    }
    LBFS_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, fn, &cfg) != cudaSuccess || ncl < 1) {
      (void)cudaGetLastError();
      continue;
    }
    if (dsm) {  // late segments of a shallow BFS run the global-claim kernel in the same launch shape
      const void* fg = (const void*)k_cluster_levels<false>;
      if (cs > 8) LBFS_CUDA(cudaFuncSetAttribute(fg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      LBFS_CUDA(cudaFuncSetAttribute(fg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    }
    cl_size_ = cs;
    cl_dsm_ = dsm;
    cl_slice_words_ = dsm ? slice : 0;
    cl_qs_ = (int32_t)qs;
    cl_mail_cap_ = (int32_t)mail_cap;
    cl_smem_ = smem;
    break;
  }
  if (!cl_size_) return;
  // a level runs on the cluster only with <= exit_edges frontier edges, so it
  // discovers at most min(exit_edges, n) vertices
  cl_cap_ = (int64_t)std::min<unsigned long long>(cl_exit_edges_, (unsigned long long)n_) + 64;
  cl_spill_ = dev_alloc<QEntry>((size_t)kMaxCluster * 2 * cl_cap_);
  cl_big_ = dev_alloc<CtaItem>((size_t)kCounterRing * cl_cap_);
  cl_big_cnt_ = dev_alloc<unsigned long long>(kCounterRing);
  LBFS_CUDA(cudaMemset(cl_big_cnt_, 0, sizeof(unsigned long long) * kCounterRing));
}

void BfsEngine::launch_cluster(int64_t L, int cur, bool prev_bitmap, cudaStream_t st, int32_t root_orig) {
  ClusterArgs p{};
  p.row_ptr = row_ptr_;
  p.col_idx = col_idx_;
  p.new2old = new2old_;
  p.old2new = old2new_;
  p.root_orig = root_orig;
  p.classes = classes_;
  p.t_cta = t_cta_;
  p.t_warp = t_warp_;
  p.t_nz = t_nz_;
  p.visited = visited_;
  p.prev = prev_;
  p.pred_int = pred_int_;
  p.level_int = level_int_;
  p.nwords = nwords_;
  p.slice_words = cl_slice_words_;
  p.qs = cl_qs_;
  p.mail_cap = cl_mail_cap_;
  p.qchunk = qchunk_;
  p.exit_warps = exit_fair_ ? expand_grid_ * (512 / 32) : 0;
  p.cap = cl_cap_;
  p.in_small = q_small_[cur];
  p.in_items = q_cta_[cur];
  if (prev_bitmap) {  // k_compact's list + warp slices + hub slices
    p.in_items2 = q_wslice_[cur];
    p.in_bitmap = 1;
  } else {  // winners' queues
    p.in_warp = q_warp_[cur];
    p.in_bitmap = 0;
  }
  p.ring = cnt_;
  p.L0 = L;
  p.max_levels = kLoopCap;
  p.exit_edges = cl_exit_edges_;
  p.exit_hub_edges = cl_exit_hub_edges_;
  p.bitmap_min_edges = (unsigned long long)std::max<int64_t>(bitmap_floor_, n_ / bitmap_div_);
  for (int b = 0; b < 2; ++b) {
    p.out_small[b] = q_small_[b];
    p.out_cta[b] = q_cta_[b];
  }
  p.spill_small = cl_spill_;
  p.big = cl_big_;
  p.big_cnt = cl_big_cnt_;
  p.layers = h_loop_layers_;
  p.mail = h_mail_;
  p.seq = h_seq_;
  p.seq_value = ++seq_;
  p.dbg = cl_dbg_;
  if (cl_prof_) {
    if (!cl_prof_buf_) cl_prof_buf_ = dev_alloc<unsigned long long>(512 + 16 * 32);
    LBFS_CUDA(cudaMemsetAsync(cl_prof_buf_, 0, sizeof(unsigned long long) * (512 + 16 * 32), st));
    p.prof = cl_prof_buf_;
    p.prof_level = cl_prof_level_;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cl_size_);
  cfg.blockDim = dim3(kClusterThreads);
  cfg.dynamicSmemBytes = cl_smem_;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cl_size_;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (behind k_init_seed / k_compact)
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  // The bitmap lives in the cluster's shared memory for a BFS's first segment
  // (nothing to load: visited = {root}) and for deep traversals (the lattice);
  // a late segment of a shallow BFS (R-MAT: the last one or two levels) claims
  // on the global bitmap instead of loading and writing back 16 slices of it
  const bool dsm = cl_dsm_ && (root_orig >= 0 || L >= 32 || cl_dsm_always_);
  if (dsm)
    LBFS_CUDA(cudaLaunchKernelEx(&cfg, k_cluster_levels<true>, p));
  else
    LBFS_CUDA(cudaLaunchKernelEx(&cfg, k_cluster_levels<false>, p));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (g_sync_each) sync_check(st, "k_cluster_levels", __FILE__, __LINE__);
  if (cl_prof_) {
    unsigned long long pr[512 + 16 * 32];
    LBFS_CUDA(cudaMemcpyAsync(pr, cl_prof_buf_, sizeof(pr), cudaMemcpyDeviceToHost, st));
    LBFS_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[lbfs] cluster L0=%lld: load %.2fus total %.2fus\n", (long long)L, (pr[1] - pr[0]) * 1e-3,
            (pr[2] - pr[0]) * 1e-3);
    for (int i = 0; i < 64 && pr[8 + 4 * i]; ++i) {
      const unsigned long long* q = pr + 8 + 4 * i;
      const unsigned long long prev_end = i ? pr[8 + 4 * (i - 1) + 3] : pr[1];
      fprintf(stderr, "[lbfs]   level %lld: loads %.2fus claims %.2fus done %.2fus sync+totals %.2fus\n",
              (long long)(L + i), q[0] ? (q[0] - prev_end) * 1e-3 : 0.0, q[1] ? (q[1] - prev_end) * 1e-3 : 0.0,
              (q[2] - prev_end) * 1e-3, (q[3] - q[2]) * 1e-3);
    }
    if (cl_prof_level_ >= 0 && pr[512]) {
      for (int w = 0; w < kClusterThreads / 32; ++w) {
        const unsigned long long* q = pr + 512 + 16 * w;
        fprintf(stderr, "[lbfs]   level %lld warp %2d:", cl_prof_level_, w);
        for (int k = 1; k < 12; ++k) fprintf(stderr, " %6.2f", q[k] ? (q[k] - pr[512]) * 1e-3 : -1.0);
        fprintf(stderr,
                "  (us after warp 0's level start: group, loads back, claims | candidates delivered, winners | accepted, "
                "expanded, cta sync, cluster sync, accept: claims back, degrees + prefetches, queue appended, "
                "expand: degrees known; each stamp costs a globaltimer read)\n");
      }
    }
  }
}

BfsEngine::~BfsEngine() {
  cudaStreamSynchronize(stream_);
  dev_free(visited_);
  dev_free(prev_);
  dev_free(stage_);
  dev_free(side_);
  dev_free(first_nbr_);
  dev_free(svmask_);
  dev_free(wmask_);
  dev_free(sdesc_);
  dev_free(pred_int_);
  dev_free(level_int_);
  dev_free(front_);
  dev_free(dense_tasks_);
  dev_free(dbg_);
  dev_free(classes_);
  dev_free(cl_spill_);
  dev_free(cl_big_);
  dev_free(cl_big_cnt_);
  dev_free(cl_prof_buf_);
  for (int b = 0; b < 2; ++b) {
    dev_free(q_small_[b]);
    dev_free(q_warp_[b]);
    dev_free(q_cta_[b]);
    dev_free(q_items_[b]);
    dev_free(q_wslice_[b]);
  }
  dev_free(cnt_);
  if (h_cnt_) cudaFreeHost(h_cnt_);
  if (h_mail_) cudaFreeHost(h_mail_);
  if (h_loop_layers_) cudaFreeHost(h_loop_layers_);
  if (out_st_) {
    cudaStreamSynchronize(out_st_);
    cudaStreamDestroy(out_st_);
    for (auto& e : ev_out_) cudaEventDestroy(e);
  }
  dev_free(own_pred_);
  dev_free(own_level_);
  for (auto& e : ev_) cudaEventDestroy(e);
  for (auto& e : ev_split_) cudaEventDestroy(e);
  cudaEventDestroy(ev_gap_);
  for (auto& e : ev_cl_) cudaEventDestroy(e);
  dev_free(row_ptr_);
  dev_free(col_idx_);
  if (new2old_loc_ != new2old_) dev_free(new2old_loc_);
  dev_free(new2old_);
  dev_free(fglob_);
  if (h_red_) cudaFreeHost(h_red_);
  dev_free(red_dev_);
  dev_free(part_err_);
  dev_free(resolve_cnt_);
  dev_free(old2new_);
  cudaStreamSynchronize(res_st_);
  cudaStreamDestroy(res_st_);
  cudaEventDestroy(ev_resolve_);
  cudaEventDestroy(ev_side_done_);
  for (auto& e : ev_snap_) cudaEventDestroy(e);
  for (auto& s : snap_) dev_free(s);
  cudaStreamDestroy(stream_);
}

void BfsEngine::ensure_own_outputs() {
  if (!own_pred_) own_pred_ = dev_alloc<int32_t>((size_t)npad_);
  if (!own_level_) own_level_ = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_, 1));
}

unsigned clamp_grid(int64_t blocks, int64_t cap) {
  return (unsigned)std::max<int64_t>(1, std::min(blocks, cap));
}

// pdl: the launch directly follows another kernel of the level on the stream
// (programmatic dependent launch: its prologue overlaps that kernel's tail)
#define LBFS_LAUNCH_EXPAND(M, P)                                                                        \
  do {                                                                                                  \
    if (pdl)                                                                                            \
      LBFS_LAUNCH_PDL((k_expand<M, P>), grid, (expand_threads<M, P>()), smem, st, a, f, hot);           \
    else                                                                                                \
      LBFS_LAUNCH((k_expand<M, P>), grid, (expand_threads<M, P>()), smem, st, a, f, hot);               \
  } while (0)

template <int M>
static void launch_expand_m(int pi, unsigned grid, int smem, const LevelArgs& a, const Frontier& f, int32_t hot,
                            cudaStream_t st, bool pdl) {
  if (pi == 0) {
    LBFS_LAUNCH_EXPAND(M, 1);
  } else if (pi == 1) {
    LBFS_LAUNCH_EXPAND(M, 2);
  } else if (pi == 3) {
    LBFS_LAUNCH_EXPAND(M, 16);
  } else if (pi == 4) {
    LBFS_LAUNCH_EXPAND(M, 32);
  } else if (pi == 5) {
    LBFS_LAUNCH_EXPAND(M, 64);
  } else if (pi == 6) {  // slice items, then the raw queues, in one launch
    if constexpr (M == kBitmapOut)
      throw Failure(LBFS_ECUDA, "internal: no fused bitmap-mode launch");
    else
      LBFS_LAUNCH_EXPAND(M, 5);
  } else {
    LBFS_LAUNCH_EXPAND(M, 4);
  }
}

void BfsEngine::launch_expand(int mode, int pi, unsigned grid, const LevelArgs& a, const Frontier& f,
                              cudaStream_t st, bool pdl) {
  if (mode == kHeavy)
    launch_expand_m<kHeavy>(pi, grid, dyn_smem_, a, f, hot_words_, st, pdl);
  else if (mode == kBitmapOut)
    launch_expand_m<kBitmapOut>(pi, grid, dyn_smem_, a, f, hot_words_, st, pdl);
  else
    launch_expand_m<kQueueOut>(pi, grid, 0, a, f, 0, st, pdl);
}

bool env_flag(const char* name) {
  const char* v = getenv(name);
  return v && *v && *v != '0';
}

LevelArgs BfsEngine::level_args() const {
  LevelArgs a{};
  a.row_ptr = row_ptr_;
  a.col_idx = col_idx_;
  a.new2old = new2old_loc_;
  a.visited = visited_;
  a.prev = prev_;
  a.pred_int = pred_int_;
  a.level_int = level_int_;
  a.classes = classes_;
  a.dbg = count_ ? dbg_ : nullptr;
  a.refresh_chunks = refresh_chunks_;
  a.t_cta = t_cta_;
  a.t_warp = t_warp_;
  a.t_nz = t_nz_;
  a.t_hub = warp_items_ ? t_warp_ : t_cta_;
  a.align_items = align_items_ ? 1 : 0;
  a.part_log = part_log_;
  a.part_rank = part_rank_;
  a.chk_n = n_;
  a.chk_nnz = nnz_loc_;
  // queue-mode hub items: small enough that a hub's row spreads over many
  // warps (a queue level is latency-bound per slice, not bandwidth-bound)
  a.qchunk = qchunk_;
  return a;
}

// A bottom-up level (bottomup.cu): the frontier bitmap (from k_compact after
// a bitmap level, else rebuilt from the queues), then one warp per visited
// word of the rows with degree >= 1. k_compact follows as for any bitmap level.
unsigned BfsEngine::bottom_up_level(const Counters& c, bool prev_bitmap, int cur, cudaStream_t st) {
  if (!prev_bitmap) {
    LBFS_CUDA(cudaMemsetAsync(front_, 0, sizeof(uint32_t) * (size_t)nwords_, st));
    const int64_t ns = (int64_t)c.bin[kBinSmall], nw = (int64_t)c.bin[kBinWarp], nc = (int64_t)c.bin[kBinCta];
    LBFS_LAUNCH(k_front_from_queues, clamp_grid((ns + nw + nc + 255) / 256, (int64_t)sm_count_ * 8), 256, 0, st,
                front_, q_small_[cur], ns, q_warp_[cur], nw, q_cta_[cur], nc, old2new_);
  }
  const int64_t nw_nz = ((int64_t)t_nz_ + 31) / 32;
  BottomUpArgs b{row_ptr_, col_idx_, new2old_loc_, front_, visited_, pred_int_, nw_nz, (int64_t)t_nz_};
  const unsigned grid = clamp_grid((nw_nz * 32 + 255) / 256, (int64_t)sm_count_ * 16);
  LBFS_LAUNCH(k_bottom_up, grid, 256, 0, st, b);
  split_any_ = false;
  return grid;
}

unsigned BfsEngine::expand_level(LevelArgs& a, const Counters& c, int mode, bool prev_bitmap, int cur, int64_t L,
                                 cudaStream_t st) {
  const bool bitmap = mode != kQueueOut;
  a.stage = stage_;
  a.stage_first = 1;
  a.stage_words = stage_words_;
  merge_words_ = hot_words_;
  a.next_level = (int32_t)(L + 1);
  a.next_cnt = &cnt_[(L + 1) % kCounterRing];
  a.next_small = q_small_[cur ^ 1];
  a.next_warp = q_warp_[cur ^ 1];
  a.next_cta = q_cta_[cur ^ 1];
  Frontier f{};
  f.cta = q_cta_[cur];
  f.n_cta = (int64_t)c.bin[kBinCta];
  if (prev_bitmap) {  // k_compact produced a list + group items
    f.list = q_small_[cur];
    f.items = q_items_[cur];
    f.n_items = (int64_t)c.bin[kBinItems];
    f.wslice = q_wslice_[cur];
    f.n_wslice = (int64_t)c.bin[kBinWSlice];
    // dense small region: stream it whole when most of it is in the frontier
    const int64_t small_region = (int64_t)t_nz_ - t_warp_;
    // (only for a large small region: below ~4 M elements streaming it whole
    // costs more than walking the list — S20 +4.5% without; S22 +1%, S24 +3% with)
    if (small_region > 0 && (int64_t)c.bin[kBinSmall] * 100 > small_region * dense_pct_ && !dense_off_ &&
        e_nz_ - e_big_ >= dense_min_elems_) {
      f.n_items = 0;
      f.front = front_;
      f.front_nc = true;
      f.dense = dense_tasks_;
      f.n_dense = n_dense_tasks_;
    }
    const int64_t warp_region = (int64_t)t_warp_ - t_cta_;
    // (opt-in: measured slower than warp slices on S24, 0.55 vs 0.36 ms)
    if (warp_region > 0 && (int64_t)c.bin[kBinWSlice] * kDenseDenom > warp_region * kDenseNum && !dense_off_ &&
        dense_warp_) {
      f.n_wslice = 0;
      f.front = front_;
      f.dense_warp = true;
    }
  } else {  // winners appended to raw queues
    f.small = q_small_[cur];
    f.warp = q_warp_[cur];
    f.n_small = (int64_t)c.bin[kBinSmall];
    f.n_warp = (int64_t)c.bin[kBinWarp];
  }
  // (a queue-mode CTA has 512 threads: one work unit per warp where the grid allows it)
  const int64_t wpc = bitmap || qgrid_old_ ? kExpandWarps : 512 / 32;
  const int64_t need = std::max({(f.n_cta + wpc - 1) / wpc, f.dense_warp ? (int64_t)1 << 30 : 0,
                                  (f.n_dense + wpc - 1) / wpc,
                                  (f.n_wslice + wpc - 1) / wpc,
                                  (f.n_items + wpc - 1) / wpc,
                                  (f.n_warp + (f.n_small + 31) / 32 + wpc - 1) / wpc,
                                  (int64_t)1});
  const unsigned grid = bitmap ? (unsigned)expand_grid_ : clamp_grid(need, expand_grid_);
  // heavy level: the whole CSR as one window stream (stream.cu): the frontier
  // bitmap (from the queues after a queue-mode level), the windows' valid
  // masks, then k_stream_heavy; no per-bin launches
  if (mode == kHeavy && stream_on_ && nparts_ == 1 && wmask_) {
    if (!prev_bitmap) {
      LBFS_CUDA(cudaMemsetAsync(front_, 0, sizeof(uint32_t) * (size_t)nwords_, st));
      const int64_t ns = (int64_t)c.bin[kBinSmall], nw = (int64_t)c.bin[kBinWarp], nc = (int64_t)c.bin[kBinCta];
      LBFS_LAUNCH(k_front_from_queues, clamp_grid((ns + nw + nc + 255) / 256, (int64_t)sm_count_ * 8), 256, 0, st,
                  front_, q_small_[cur], ns, q_warp_[cur], nw, q_cta_[cur], nc, old2new_);
    }
    const int64_t nsw = svmask_ ? n_win_all_ - w_small0_ : 0;
    if (nsw > 0)
      LBFS_LAUNCH(k_sweep_plan_small, (unsigned)((nsw + 63) / 64), 256, 0, st, classes_, sdesc_, front_, e_nz_,
                  w_small0_, nsw, svmask_);
    LBFS_LAUNCH(k_window_masks, clamp_grid((n_side_win_ + 255) / 256, (int64_t)sm_count_ * 8), 256, 0, st, side_,
                n_side_win_, e_big_, front_, nsw > 0 ? svmask_ : nullptr, w_small0_, wmask_);
    StreamArgs sa{col_idx_, wmask_, svmask_, n_win_all_, n_side_win_, w_small0_, visited_, stage_, stage_words_,
                  stream_hot_words_};
    LBFS_LAUNCH(k_stream_heavy<kStreamDepth>, (unsigned)sm_count_, kStreamThreads, stream_hot_words_ * 4, st, sa);
    merge_words_ = stream_hot_words_;
    sweep_used_ = true;
    split_any_ = true;
    return (unsigned)sm_count_;
  }
  // heavy level after a bitmap level: the big-row region is swept whole (sweep.cu)
  // (only when the frontier's big rows hold enough of the region's edges:
  // below that the sweep streams mostly rows outside the frontier)
  // after a queue-mode level (opt-in experiment, LBFS_SWEEP_AFTER_QUEUE): the
  // frontier bitmap is rebuilt from the queues and the hub + warp-bin rows
  // (the big-row region) are swept; the small queue keeps its own launch
  const bool from_queues = mode == kHeavy && !prev_bitmap && sweep_after_queue_ && nparts_ == 1;
  const bool sweep = mode == kHeavy && (prev_bitmap || from_queues) && side_ && sweep_fits_ &&
                     !sweep_off_ &&
                     (from_queues ||
                      c.big_edges * 100ull >= (unsigned long long)e_big_ * (unsigned long long)sweep_min_pct_);
  if (sweep && from_queues) {
    LBFS_CUDA(cudaMemsetAsync(front_, 0, sizeof(uint32_t) * (size_t)nwords_, st));
    const int64_t nw = (int64_t)c.bin[kBinWarp], nc = (int64_t)c.bin[kBinCta];
    LBFS_LAUNCH(k_front_from_queues, clamp_grid((nw + nc + 255) / 256, (int64_t)sm_count_ * 8), 256, 0, st, front_,
                q_small_[cur], 0, q_warp_[cur], nw, q_cta_[cur], nc, old2new_);
    f.n_warp = 0;  // (the warp-bin rows are in the swept region)
  }
  sweep_used_ = sweep;
  if (sweep) merge_words_ = sweep_hot_words_;
  if (sweep) {
    if (split_) LBFS_CUDA(cudaEventRecord(ev_split_[0], st));
    // (window infos are computed by the sweep's producers from the side entries and front_)
    // the small region joins the sweep when most of it is in the frontier
    // (else its frontier rows go through the group items below)
    const bool sweep_small = svmask_ && f.n_dense > 0 && sweep_small_;
    if (sweep_small) {
      const int64_t nsw = n_win_all_ - w_small0_;
      LBFS_LAUNCH(k_sweep_plan_small, (unsigned)((nsw + 63) / 64), 256, 0, st, classes_, sdesc_, front_, e_nz_,
                  w_small0_, nsw, svmask_);
    }
    SweepArgs sa{col_idx_, side_, n_side_win_, e_big_, sweep_small ? n_win_all_ : n_side_win_,
                 sweep_small ? e_nz_ : e_big_, sweep_small ? w_small0_ : n_win_all_ + 1, svmask_, front_,
                 visited_, pred_int_, new2old_loc_,
                 stage_, 1, stage_words_, sweep_hot_words_, getenv("LBFS_SWEEP_PF") ? atoi(getenv("LBFS_SWEEP_PF")) : kSweepPrefetch,
                 getenv("LBFS_SWEEP_DBG") ? atoi(getenv("LBFS_SWEEP_DBG")) : 0, nullptr, 0, classes_};
    // the dense small region rides along on the sweep's worker warps
    if (f.n_dense > 0 && !sweep_small && sweep_workers_ && kSweepWorkers > 0) {
      sa.dense = f.dense;
      sa.n_dense = f.n_dense;
      f.n_dense = 0;
    }
    LBFS_LAUNCH(k_sweep, (unsigned)expand_grid_, kSweepThreads, kSweepRingBytes + sweep_hot_words_ * 4, st, sa);
    a.stage_first = 0;
    f.n_cta = 0;
    f.n_wslice = 0;
    f.dense_warp = false;
    if (sweep_small) {  // the small region is swept too
      f.n_items = 0;
      f.n_dense = 0;
    }
  }
  const bool any = f.n_cta + f.n_warp + f.n_small + f.n_items + f.n_wslice + f.n_dense > 0 || f.dense_warp;
  if (any) {
    // one launch per non-empty bin: each phase kernel gets its own register
    // allocation (the fused kernel was capped at 64 registers by 1024 threads)
    bool has[6] = {f.n_cta > 0, f.n_items > 0, f.n_warp + f.n_small > 0, f.n_wslice > 0, f.n_dense > 0,
                   f.dense_warp};
    // after a queue-mode level the frontier is slice items + raw queues: one
    // launch for both (a launch costs ~5-10 us here: a queue level is short,
    // a heavy launch zeroes and stores its hot rows)
    bool follows = sweep && !split_;  // a kernel of this level is already on the stream
    if (fuse_queues_ && !prev_bitmap && mode != kBitmapOut && has[0] && has[2] && !split_) {
      launch_expand(mode, 6, grid, a, f, st, follows);
      a.stage_first = 0;
      has[0] = has[2] = false;
      follows = true;
    }
    for (int pi = 0; pi < 6; ++pi) {
      if (split_ && !(sweep && pi == 0)) LBFS_CUDA(cudaEventRecord(ev_split_[pi], st));
      if (!has[pi]) continue;
      launch_expand(mode, pi, grid, a, f, st, follows);
      a.stage_first = 0;
      follows = !split_;
    }
    if (split_) LBFS_CUDA(cudaEventRecord(ev_split_[6], st));
  }
  split_any_ = any || sweep;
  return grid;
}

void BfsEngine::compact_level(int cur, int64_t L, uint32_t* fsend, cudaStream_t st, bool heavy, bool pdl) {
  CompactArgs ca{row_ptr_, new2old_loc_, visited_, prev_, nwl_, level_int_, (int32_t)(L + 1),
                 t_cta_, t_warp_, t_nz_, &cnt_[(L + 1) % kCounterRing], q_small_[cur ^ 1], q_cta_[cur ^ 1],
                 q_items_[cur ^ 1], q_wslice_[cur ^ 1], front_, part_log_, part_rank_, fsend,
                 col_idx_, first_nbr_, pred_int_,
                 0,  // heavy: blind ORs leave no parent; k_resolve gives them one off the critical path
                 (int32_t)L};
  const bool small_graph = n_loc_ < kCompactSmallGraph && !compact_big_;
  const int cv = small_graph ? kCompactVertsSmall : kCompactVertsBig;
  const unsigned cgrid = (unsigned)((n_loc_ + cv - 1) / cv);
  if (small_graph) {
    if (pdl)
      LBFS_LAUNCH_PDL(k_compact<kCompactVertsSmall>, cgrid, kCompactThreads, 0, st, ca);
    else
      LBFS_LAUNCH(k_compact<kCompactVertsSmall>, cgrid, kCompactThreads, 0, st, ca);
  } else {
    if (pdl)
      LBFS_LAUNCH_PDL(k_compact<kCompactVertsBig>, cgrid, kCompactThreads, 0, st, ca);
    else
      LBFS_LAUNCH(k_compact<kCompactVertsBig>, cgrid, kCompactThreads, 0, st, ca);
  }
  if (heavy && lean_events_ && nparts_ == 1) {
    resolve_deferred_ = L + 1;  // (launched behind the level's publish / cluster kernel: launch_resolve)
    return;
  }
  if (heavy) launch_resolve(L + 1, st);
}

// (lean events) the side work of the level just launched, behind its publish /
// cluster kernel on the stream and before the host waits for the mailbox
void BfsEngine::flush_resolve(cudaStream_t st) {
  if (resolve_deferred_ < 0) return;
  launch_resolve(resolve_deferred_, st);
  resolve_deferred_ = -1;
}

// The parents of a heavy level's new vertices (level lvl) are read by
// k_finalize only: resolve them on the side stream while the next levels run
// (joined before k_finalize).
void BfsEngine::launch_resolve(int64_t lvl, cudaStream_t st) {
  const int64_t L = lvl - 1;
  {
    LBFS_CUDA(cudaEventRecord(ev_resolve_, st));
    LBFS_CUDA(cudaStreamWaitEvent(res_st_, ev_resolve_, 0));
    const int64_t n4 = (n_loc_ + 3) / 4;
    // (short blocks, no grid-stride clamp: a block that lives for the whole
    // kernel would keep the next level's one-CTA-per-SM kernels off its SM)
    cudaStream_t rs = resolve_inline_ ? st : res_st_;
    LBFS_LAUNCH(k_resolve, resolve_clamp_ ? clamp_grid((n4 + 255) / 256, (int64_t)sm_count_ * 16)
                                          : (unsigned)((n4 + 255) / 256),
                256, 0, rs, level_int_, first_nbr_, row_ptr_, col_idx_, new2old_loc_, pred_int_, n_loc_,
                (int32_t)(L + 1));
    side_pending_ = true;
  }
}

// Parents of the vertices at level lvl (found by blind ORs at a heavy level):
// the first neighbour one level up; rows are sorted by internal id, i.e. by
// descending degree, and the first entry is almost always it (else scan on).
// Any such neighbour is a valid parent (traversal.py:145-147).
__global__ void __launch_bounds__(256) k_resolve(const int32_t* level_int,
                                                 const int32_t* __restrict__ first_nbr,
                                                 const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                                                 const int32_t* __restrict__ new2old, int32_t* __restrict__ pred_int,
                                                 int64_t n, int32_t lvl) {
  const int64_t n4 = (n + 3) / 4;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    // (plain loads, not the read-only path: later levels keep writing
    // level_int while this runs on the side stream; the entries compared here
    // were written before it, and a concurrent write only ever stores a level
    // above lvl, so a stale view cannot make a wrong match)
    const int4 l4 = reinterpret_cast<const int4*>(level_int)[i];  // (level_int is padded to 4)
    const int32_t lv4[4] = {l4.x, l4.y, l4.z, l4.w};
    bool need[4];
    int32_t u[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      need[q] = lv4[q] == lvl && 4 * i + q < n;
      u[q] = need[q] ? __ldg(first_nbr + 4 * i + q) : 0;
    }
    int32_t lu[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) lu[q] = need[q] ? level_int[u[q]] : 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!need[q]) continue;
      const int64_t v = 4 * i + q;
      int32_t par = kSentinel;
      if (lu[q] == lvl - 1) {
        par = __ldg(new2old + u[q]);
      } else {
        const int64_t e = __ldg(row_ptr + v + 1);
        for (int64_t k = __ldg(row_ptr + v) + 1; k < e; ++k) {
          const int32_t x = __ldg(col_idx + k);
          if (level_int[x] == lvl - 1) {
            par = __ldg(new2old + x);
            break;
          }
        }
      }
      pred_int[v] = par;
    }
  }
}

void BfsEngine::merge_hot(cudaStream_t st) {
  // (the sweep stores whole rows first in its level; expand kernels alone write only their prefix)
  const int hw4 = merge_words_ / 4;
  const dim3 grid((unsigned)((hw4 + 255) / 256), (unsigned)((expand_grid_ + kMergeRows - 1) / kMergeRows));
  // (directly behind the level's last expansion kernel)
  if (split_)
    LBFS_LAUNCH(k_merge_hot, grid, 256, 0, st, reinterpret_cast<const uint4*>(stage_), expand_grid_, hw4,
                stage_words_ / 4, visited_);
  else
    LBFS_LAUNCH_PDL(k_merge_hot, grid, 256, 0, st, reinterpret_cast<const uint4*>(stage_), expand_grid_, hw4,
                    stage_words_ / 4, visited_);
}

// Output pass: parents (pad32(n), SENTINEL padding) and, when asked for,
// levels in original ids. With host_pred_ set, the parents are produced in
// kOutChunks pieces and each piece is copied to the host on out_st_ as soon
// as it is written, so the D2H overlaps the rest of the pass.
void BfsEngine::finalize(int32_t* d_pred, int32_t* d_level, cudaStream_t st) {
  const bool vec = ((uintptr_t)d_pred % 16) == 0;
  const int64_t chunks = host_pred_ ? kOutChunks : 1;
  const int64_t step = (npad_ / chunks + 31) / 32 * 32;
  for (int64_t x0 = 0, k = 0; x0 < npad_; x0 += step, ++k) {
    const int64_t x1 = std::min(npad_, x0 + step);
    const unsigned grid = clamp_grid(((x1 - x0) / 4 + 255) / 256, (int64_t)sm_count_ * 8);
    if (vec)
      LBFS_LAUNCH(k_finalize<true>, grid, 256, 0, st, old2new_, visited_, pred_int_, kSentinel, n_, x0, x1, d_pred);
    else
      LBFS_LAUNCH(k_finalize<false>, grid, 256, 0, st, old2new_, visited_, pred_int_, kSentinel, n_, x0, x1, d_pred);
    if (host_pred_) {
      LBFS_CUDA(cudaEventRecord(ev_out_[k], st));
      LBFS_CUDA(cudaStreamWaitEvent(out_st_, ev_out_[k], 0));
      LBFS_CUDA(cudaMemcpyAsync(host_pred_ + x0, d_pred + x0, sizeof(int32_t) * (size_t)(x1 - x0),
                                cudaMemcpyDeviceToHost, out_st_));
    }
  }
  if (d_level) levels_out(d_level, st);
}

void BfsEngine::levels_out(int32_t* d_level, cudaStream_t st) {
  const bool vec = ((uintptr_t)d_level % 16) == 0;
  const unsigned grid = clamp_grid((n_ / 4 + 255) / 256, (int64_t)sm_count_ * 8);
  if (vec)
    LBFS_LAUNCH(k_finalize<true>, grid, 256, 0, st, old2new_, visited_, level_int_, -1, n_, 0, n_, d_level);
  else
    LBFS_LAUNCH(k_finalize<false>, grid, 256, 0, st, old2new_, visited_, level_int_, -1, n_, 0, n_, d_level);
}

// BFS with host outputs (lbfs_bfs): parents copied chunk by chunk behind the
// output pass; levels (optional) after it.
void BfsEngine::run_to_host(int64_t root, int direction, int32_t* h_pred, int32_t* h_level, lbfs_timing* t) {
  ensure_own_outputs();
  if (!out_st_) {
    LBFS_CUDA(cudaStreamCreateWithFlags(&out_st_, cudaStreamNonBlocking));
    for (auto& e : ev_out_) LBFS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  host_pred_ = h_pred;
  const auto t0 = std::chrono::steady_clock::now();
  try {
    run(root, own_pred_, h_level ? own_level_ : nullptr, t, direction);
  } catch (...) {
    host_pred_ = nullptr;
    cudaStreamSynchronize(out_st_);
    throw;
  }
  host_pred_ = nullptr;
  if (h_level)
    LBFS_CUDA(cudaMemcpyAsync(h_level, own_level_, sizeof(int32_t) * (size_t)n_, cudaMemcpyDeviceToHost, out_st_));
  LBFS_CUDA(cudaStreamSynchronize(out_st_));
  if (t) {  // host wall time of the copies that did not overlap the BFS
    const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    t->d2h_ms = std::max(0.0, wall - t->bfs_ms);
  }
}

void BfsEngine::last_levels_to_host(int32_t* h_level) {
  ensure_own_outputs();
  levels_out(own_level_, stream_);
  LBFS_CUDA(cudaMemcpyAsync(h_level, own_level_, sizeof(int32_t) * (size_t)n_, cudaMemcpyDeviceToHost, stream_));
  LBFS_CUDA(cudaStreamSynchronize(stream_));
}

// Tuning / debug switches, read once per graph handle (not per BFS).
void BfsEngine::read_env() {
  auto geti = [](const char* name, long long dflt) {
    const char* v = getenv(name);
    return v && *v ? atoll(v) : dflt;
  };
  trace_ = env_flag("LBFS_TRACE");   // per-level table on stderr (the GPU analogue of scripts/layer_profile.py)
  split_ = env_flag("LBFS_SPLIT");   // one launch per bin, timed separately
  count_ = env_flag("LBFS_COUNT");   // candidate-write counters (slow)
  part_heavy_off_ = geti("LBFS_PART_HEAVY", 1) == 0;
  part_sparse_mode_ = (int)geti("LBFS_PART_SPARSE", 1);
  bu_alpha_ = (int)std::max<long long>(1, geti("LBFS_BU_ALPHA", 14));
  bu_beta_ = (int)std::max<long long>(1, geti("LBFS_BU_BETA", 24));
  bitmap_div_ = (int)std::max<long long>(1, geti("LBFS_BITMAP_DIV", kBitmapDiv));  // bitmap mode from n / this edges
  bitmap_floor_ = std::max<long long>(1, geti("LBFS_BITMAP_MIN", (long long)1 << 16));
  sweep_min_pct_ = (int)geti("LBFS_SWEEP_MIN", kSweepMinPct);
  heavy_div_ = (int)geti("LBFS_HEAVY_DIV", kHeavyDiv);  // heavy (blind-OR) from nnz / this edges (0: off)
  heavy_vis_pct_ = (int)geti("LBFS_HEAVY_VIS", 0);     // ... while visited edge mass <= this % of the frontier's (0: off)
  dense_off_ = env_flag("LBFS_NO_DENSE");
  dense_pct_ = (int)geti("LBFS_DENSE_PCT", 100 * kDenseNum / kDenseDenom);
  dense_min_elems_ = geti("LBFS_DENSE_MIN", kDenseMinElems);
  dense_warp_ = env_flag("LBFS_DENSE_WARP");
  sweep_off_ = env_flag("LBFS_NO_SWEEP");
  stream_on_ = geti("LBFS_STREAM", 0) != 0;  // (experiment: the full-CSR window stream; slower today)
  sweep_after_queue_ = env_flag("LBFS_SWEEP_AFTER_QUEUE");
  sweep_small_ = env_flag("LBFS_SWEEP_SMALL");
  refresh_chunks_ = (int)geti("LBFS_REFRESH", kRefreshChunks);
  qchunk_ = (int)std::min<long long>(kChunk, std::max<long long>(kQChunkMin, geti("LBFS_QCHUNK", kQChunkDefault))) & ~127;
  // small-frontier levels run on the cluster while a frontier has at most this many edges
  cl_exit_edges_ = (unsigned long long)std::max<long long>(64, geti("LBFS_CLUSTER_EDGES", kClusterExitEdges));
  cl_exit_hub_edges_ = (unsigned long long)std::max<long long>(64, geti("LBFS_CLUSTER_HUB_EDGES", kClusterExitHubEdges));
  cl_mail_cap_env_ = (int)geti("LBFS_CLUSTER_MAIL_CAP", 0);
  cl_no_mail_ = env_flag("LBFS_CLUSTER_NO_MAIL");  // (A/B) DSMEM mode with remote claims instead of candidate mailboxes
  cl_no_dsm_ = env_flag("LBFS_CLUSTER_GLOBAL");  // claim on the global bitmap even when the slices fit
  cl_off_ = env_flag("LBFS_NO_CLUSTER");
  // queue-mode winners emit warp-bin rows as slice items (S24 379 -> 385 GTEPS);
  // LBFS_NO_WARP_ITEMS=1: append them to the raw warp queue instead
  warp_items_ = !env_flag("LBFS_NO_WARP_ITEMS");
  qgrid_old_ = env_flag("LBFS_QGRID_OLD");
  compact_big_ = env_flag("LBFS_COMPACT_BIG");  // (A/B) 4096-id compaction blocks on small graphs too
  // No timing events between the kernels of a BFS: an event record between two
  // kernels costs a few microseconds of stream serialisation each and ends a
  // chain of programmatic dependent launches (S24 401 -> 414, S20 106 -> 117
  // GTEPS). The cluster segments report their own device time through the
  // mailbox; LBFS_FULL_EVENTS=1 (and the trace modes) bracket every level.
  lean_events_ = !env_flag("LBFS_FULL_EVENTS") && !trace_ && !split_;
  align_items_ = env_flag("LBFS_ALIGN_ITEMS");  // (A/B) queue-mode winners cut their slice items on window boundaries
  sweep_workers_ = !env_flag("LBFS_NO_SWEEP_WORKERS");  // (A/B) the dense small region as its own launch
  cl_dsm_always_ = env_flag("LBFS_CLUSTER_DSM_ALWAYS");  // (A/B) every cluster segment with the bitmap in DSMEM
  exit_fair_ = !env_flag("LBFS_NO_EXIT_FAIR");  // (A/B) cluster exit items of qchunk edges whatever the frontier
  fuse_queues_ = !env_flag("LBFS_NO_FUSE_QUEUES");  // (A/B) one launch per bin after a queue-mode level
  publish_after_heavy_ = !env_flag("LBFS_NO_PUBLISH_AFTER_HEAVY");  // (A/B) always hand the next frontier to the cluster
  resolve_inline_ = env_flag("LBFS_RESOLVE_INLINE");  // (A/B) k_resolve on the level stream
  resolve_clamp_ = env_flag("LBFS_RESOLVE_CLAMP");    // (A/B) k_resolve as a clamped grid-stride grid  // (A/B) size queue-mode grids for 32 warps per CTA
  cl_prof_ = env_flag("LBFS_CLUSTER_PROF");
  cl_force_size_ = (int)geti("LBFS_CLUSTER_SIZE", 0);  // (experiment) 2, 4, 8 or 16
  cl_dbg_ = (int)geti("LBFS_CLUSTER_DBG", 0);
  cl_prof_level_ = geti("LBFS_CLUSTER_PROF_LEVEL", -1);
}

void BfsEngine::run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t, int direction) {
  if (root < 0 || root >= n_) throw_inval("root out of range");
  if (nparts_ != 1) throw_inval("partitioned graph: use the lbfs_part_* level steps");
  if (direction != 0 && direction != 1) throw_inval("unknown direction");
  cudaStream_t st = stream_;
  if (side_pending_) {  // an earlier run failed after launching side work: let it finish first
    cudaStreamSynchronize(res_st_);
    side_pending_ = false;
  }
  const int64_t launches0 = g_launches.load();
  n_cl_ev_ = 0;
  resolve_deferred_ = -1;
  LBFS_CUDA(cudaEventRecord(ev_[0], st));
  LevelArgs a = level_args();
  a.next_small = q_small_[0];
  a.next_warp = q_warp_[0];
  a.next_cta = q_cta_[0];
  {  // K4: bitmaps + internal levels + counter ring + the root (outputs are written once, by k_finalize)
    const unsigned grid = clamp_grid((n_ / 4 + 255) / 256, (int64_t)sm_count_ * 8);
    LBFS_LAUNCH(k_init_seed, grid, 256, 0, st, (uint4*)visited_, (uint4*)prev_, (nwords_ + 3) / 4, (int4*)level_int_,
                (n_ + 3) / 4, cnt_, a, old2new_, (int32_t)root);
  }
  if (!lean_events_) LBFS_CUDA(cudaEventRecord(ev_[1], st));
  const bool use_cluster = cl_size_ > 0 && !cl_off_ && !split_ && !count_;
  if (!use_cluster) {
    LBFS_CUDA(cudaMemcpyAsync(h_mail_, &cnt_[0], sizeof(Counters), cudaMemcpyDeviceToHost, st));
    LBFS_CUDA(cudaStreamSynchronize(st));
  }
  layers_.clear();
  double expand_ms = 0.0, cluster_ms = 0.0;
  bool prev_bitmap = false, prev_bu = false, timed_level = false;
  bool expect_big = false;  // the level just launched was heavy: its output is published by k_publish
  const unsigned long long bitmap_min_edges = (unsigned long long)std::max<int64_t>(bitmap_floor_, n_ / bitmap_div_);
  int64_t L = 0;
  int cur = 0;  // queue parity == L & 1
  bool pending = false;  // the layer of the last full-GPU level waits for the next frontier's size
  lbfs_layer pend{};
  for (;;) {
    // (1) small-frontier levels on the cluster; its mailbox also carries the
    // counters of the frontier a full-GPU level just produced
    Counters c{};
    int64_t k = 0;
    bool small_next = true;
    if (use_cluster && expect_big) {
      // after a heavy level the next frontier is almost never small: a one-warp
      // publish kernel instead of a 16-CTA cluster launch that would only
      // publish (the cluster follows when the frontier is small after all)
      publish_and_wait((int)(L % kCounterRing), (int)((L + 1) % kCounterRing), st);
      c = h_cnt_[L % kCounterRing];
      small_next = c.discovered > 0 && cluster_takes(c.discovered, c.edges, cl_exit_edges_, cl_exit_hub_edges_);
    }
    if (use_cluster && small_next) {
      const int ce = !lean_events_ && n_cl_ev_ < kClEvents ? n_cl_ev_++ : -1;
      if (ce >= 0) LBFS_CUDA(cudaEventRecord(ev_cl_[2 * ce], st));
      launch_cluster(L, cur, prev_bitmap, st, L == 0 ? (int32_t)root : -1);
      if (ce >= 0) LBFS_CUDA(cudaEventRecord(ev_cl_[2 * ce + 1], st));
      flush_resolve(st);
      wait_mail(seq_, st);
      std::atomic_thread_fence(std::memory_order_acquire);
      c = *const_cast<const Counters*>(h_mail_);
      if (lean_events_) cluster_ms += 1e-6 * (double)const_cast<volatile unsigned long long*>(h_seq_)[1];
      k = (int64_t)c.pad[0] - L;
      if (k < 0 || k > kLoopCap) throw Failure(LBFS_ECUDA, "internal: cluster level loop state");
    } else if (use_cluster) {
      // (published above)
    } else if (L == 0) {
      c = *const_cast<const Counters*>(h_mail_);
    } else {
      publish_and_wait((int)(L % kCounterRing), (int)((L + 1) % kCounterRing), st);
      c = h_cnt_[L % kCounterRing];
    }
    if (timed_level && !lean_events_) {  // the last full-GPU level's expansion (its events completed before the mailbox)
      float ms = 0.f;
      LBFS_CUDA(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
      expand_ms += ms;
      timed_level = false;
    }
    if (pending) {
      pend.discovered = k > 0 ? h_loop_layers_[0].input : (int64_t)c.discovered;
      layers_.push_back(pend);
      pending = false;
    }
    if (k > 0) {
      for (int64_t i = 0; i < k; ++i) layers_.push_back(h_loop_layers_[i]);
      if (trace_)
        fprintf(stderr, "[lbfs] L%-3lld..L%-3lld cluster (%lld levels), next in=%llu edges=%llu\n", (long long)L,
                (long long)(L + k - 1), (long long)k, c.discovered, c.edges);
      L += k;
      cur = (int)(L & 1);
      prev_bitmap = prev_bu = false;
    }
    if (c.discovered == 0) break;
    if (k > 0 && cluster_takes(c.discovered, c.edges, cl_exit_edges_, cl_exit_hub_edges_)) continue;  // the cluster stopped at its level cap
    // (2) one level on the whole GPU
    const bool bitmap = c.edges >= bitmap_min_edges;
    // direction-optimising (opt-in): bottom-up while the frontier's edges
    // outweigh the unvisited vertices' edges / alpha, back to top-down when
    // the frontier drops below n / beta (Beamer et al.'s rule)
    bool bottom_up = false;
    if (direction && bitmap) {
      unsigned long long seen = c.edges;  // degrees of every vertex visited so far (each was one frontier)
      for (const auto& l : layers_) seen += (unsigned long long)l.edges;
      const unsigned long long m_u = (unsigned long long)nnz_ > seen ? (unsigned long long)nnz_ - seen : 0ull;
      bottom_up = prev_bu ? c.discovered * (unsigned long long)bu_beta_ >= (unsigned long long)n_
                          : c.edges * (unsigned long long)bu_alpha_ > m_u;
    }
    // heavy (blind-OR) semantics pay off while most targets are unvisited:
    // the edge mass of the vertices visited before this frontier (each was
    // one frontier once) stays below heavy_vis_pct_ % of the frontier's own
    unsigned long long seen_before = 0;
    for (const auto& l : layers_) seen_before += (unsigned long long)l.edges;
    const bool heavy = !bottom_up && bitmap && stage_ && heavy_div_ > 0 &&
                       c.edges * (unsigned long long)heavy_div_ >= (unsigned long long)nnz_ &&
                       (heavy_vis_pct_ <= 0 || seen_before * 100ull <= c.edges * (unsigned long long)heavy_vis_pct_);
    if (!lean_events_) LBFS_CUDA(cudaEventRecord(ev_[2], st));
    const unsigned grid = bottom_up ? bottom_up_level(c, prev_bitmap, cur, st)
                                    : expand_level(a, c, heavy ? kHeavy : bitmap ? kBitmapOut : kQueueOut, prev_bitmap,
                                                   cur, L, st);
    if (heavy) merge_hot(st);
    // the level's kernels (expansion, merge, compaction) follow one another
    // directly on the stream (programmatic dependent launches); the timing
    // event closes the level behind the compaction (trace modes: before it)
    const bool ev_mid = (trace_ || split_ || bottom_up) && !lean_events_;
    if (ev_mid) LBFS_CUDA(cudaEventRecord(ev_[3], st));
    timed_level = true;
    if (bitmap) compact_level(cur, L, nullptr, st, heavy, !ev_mid);
    if (!ev_mid && !lean_events_) LBFS_CUDA(cudaEventRecord(ev_[3], st));
    if (trace_ || split_) {
      LBFS_CUDA(cudaEventRecord(ev_[5], st));
      LBFS_CUDA(cudaEventSynchronize(ev_[5]));
      float ms = 0.f, cms = 0.f;
      LBFS_CUDA(cudaEventElapsedTime(&ms, ev_[2], ev_[3]));
      LBFS_CUDA(cudaEventElapsedTime(&cms, ev_[3], ev_[5]));
      fprintf(stderr,
              "[lbfs] L%-3lld %s in=%-9llu edges=%-10llu big=%-10llu bins(s|list/w/c/items/ws)=%llu/%llu/%llu/%llu/%llu "
              "grid=%u expand=%.3fms compact=%.3fms\n",
              (long long)L, bottom_up ? "bottom" : heavy ? (sweep_used_ ? "sweep " : "heavy ") : bitmap ? "bitmap" : "queue ",
              c.discovered, c.edges, c.big_edges, c.bin[0], c.bin[1], c.bin[2], c.bin[3], c.bin[4], grid, ms,
              bitmap ? cms : 0.f);
      if (split_ && split_any_) {
        float sm[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int pi = 0; pi < 6; ++pi) LBFS_CUDA(cudaEventElapsedTime(&sm[pi], ev_split_[pi], ev_split_[pi + 1]));
        fprintf(stderr, "[lbfs]      split: hub=%.3fms items=%.3fms queues=%.3fms wslice=%.3fms dense=%.3fms dwarp=%.3fms\n",
                sm[0], sm[1], sm[2], sm[3], sm[4], sm[5]);
      }
    }
    if (count_) {
      unsigned long long dbg[4] = {0, 0, 0, 0};
      LBFS_CUDA(cudaMemcpy(dbg, dbg_, sizeof(dbg), cudaMemcpyDeviceToHost));
      LBFS_CUDA(cudaMemset(dbg_, 0, sizeof(dbg)));
      fprintf(stderr, "[lbfs]      candidate writes hot=%llu cold=%llu streamed elements=%llu dwarp rows=%llu\n",
              dbg[0], dbg[1], dbg[2], dbg[3]);
    }
    // ... or a level of the growth phase (its frontier has 8x the edges of the one before)
    const unsigned long long before_edges = layers_.empty() ? 0ull : (unsigned long long)layers_.back().edges;
    expect_big = publish_after_heavy_ && (heavy || (!bottom_up && c.edges >= 8ull * before_edges));
    pend = lbfs_layer{(int64_t)c.discovered, (int64_t)c.edges, 0};
    pending = true;
    cur ^= 1;
    ++L;
    prev_bitmap = bitmap;
    prev_bu = bottom_up;
  }
  if (side_pending_) {  // parents resolved on the side stream
    LBFS_CUDA(cudaEventRecord(ev_side_done_, res_st_));
    LBFS_CUDA(cudaStreamWaitEvent(st, ev_side_done_, 0));
    side_pending_ = false;
  }
  LBFS_CUDA(cudaEventRecord(ev_[6], st));
  finalize(d_pred, d_level, st);
  LBFS_CUDA(cudaEventRecord(ev_[4], st));
  LBFS_CUDA(cudaEventSynchronize(ev_[4]));
  for (int i = 0; i < n_cl_ev_; ++i) {  // cluster segments
    float ms = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&ms, ev_cl_[2 * i], ev_cl_[2 * i + 1]));
    cluster_ms += ms;
  }
  if (trace_) {
    float fin = 0.f, tot = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&fin, ev_[6], ev_[4]));
    LBFS_CUDA(cudaEventElapsedTime(&tot, ev_[0], ev_[4]));
    fprintf(stderr, "[lbfs] cluster %.3fms finalize %.3fms total %.3fms\n", cluster_ms, fin, tot);
  }
  if (t) {
    float total = 0.f, init = 0.f, fin = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&total, ev_[0], ev_[4]));
    if (!lean_events_) LBFS_CUDA(cudaEventElapsedTime(&init, ev_[0], ev_[1]));
    LBFS_CUDA(cudaEventElapsedTime(&fin, ev_[6], ev_[4]));
    if (lean_events_) {  // everything before the output pass that is not a cluster segment
      float loop = 0.f;
      LBFS_CUDA(cudaEventElapsedTime(&loop, ev_[0], ev_[6]));
      expand_ms = std::max(0.0, (double)loop - cluster_ms);
    }
    t->bfs_ms = total;
    t->init_ms = init;
    t->expand_ms = expand_ms;
    t->cluster_ms = cluster_ms;
    t->finalize_ms = fin;
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
