// BFS engine: device layout of one graph and the level driver.
//
// Layout (built once per graph): vertices are relabelled in
// descending-degree order ("internal ids"). The visited bitmap, frontier
// bins and the traversal CSR use internal ids; predecessor and level outputs
// are written in the caller's (original) ids through new2old. With this
// order the degree bins are id ranges and the visited words of the hubs —
// the targets of most probes in a power-law graph — are a small prefix of
// the bitmap that stays resident in L1.
#pragma once

#include "lbfs_internal.cuh"

namespace lbfs {

constexpr int32_t kSentinel = LBFS_SENTINEL;  // traversal.py:22
constexpr int kSmallMax = 32;                 // deg < 32: warp-cooperative small bin
constexpr int kCtaMin = 1024;                 // deg >= 1024: CTA bin (TMA-staged chunks)
constexpr int kQChunkMin = 128;              // smallest queue-mode hub item (sizes the item buffers)
#ifndef LBFS_QCHUNK_DEFAULT
#define LBFS_QCHUNK_DEFAULT 512
#endif
constexpr int kQChunkDefault = LBFS_QCHUNK_DEFAULT;  // default queue-mode hub item (LBFS_QCHUNK overrides)
constexpr int kChunk = 3968;                  // edges per CTA-bin item (31 windows of 128)
constexpr int kBinSmall = 0, kBinWarp = 1, kBinCta = 2, kBinItems = 3, kBinWSlice = 4;
constexpr int kItemElems = 512;               // elements per group item (load balance unit)
constexpr int kCounterRing = 3;
#ifndef LBFS_EXPAND_WARPS
#define LBFS_EXPAND_WARPS 32
#endif
constexpr int kExpandWarps = LBFS_EXPAND_WARPS;
constexpr int kExpandThreads = 32 * kExpandWarps;
constexpr int kRefreshChunks = 4;                 // hub chunks (warp 0) between snapshot refreshes

// Per-level counters (K6). Slot L holds the frontier of level L:
// discovered = |frontier| (layers[L].input), edges = sum of its degrees
// (layers[L].edges); bin[] are the bin sizes (entries / items).
// Expansion modes (bfs.cu): bitmap-mode output, queue-mode output, queue mode
// inside the device loop, heavy (blind-OR) bitmap levels.
enum Mode : int { kBitmapOut = 0, kQueueOut = 1, kQueueDirect = 2, kHeavy = 3 };

struct alignas(64) Counters {
  unsigned long long bin[5];  // small queue | small list, warp queue, hub slices, group items, warp slices
  unsigned long long discovered;
  unsigned long long edges;
  unsigned long long pad[1];       // (mailbox copy of k_levels: the level it stopped at)
  unsigned long long big_edges;    // bitmap-mode frontier: edges of its rows with degree >= 32 (the sweep region)
};

// A balanced unit of non-hub work: up to 32 consecutive entries of the
// frontier list (ascending internal ids) and the element range [elo, ehi)
// of their concatenated rows.
struct alignas(8) GroupItem {
  int64_t list_start;
  int32_t count;
  int32_t elo, ehi;
  int32_t pad;
};

struct alignas(16) CtaItem {  // one kChunk-edge slice of a hub's row
  int64_t start;   // absolute col_idx offset of the slice
  int32_t len;     // <= kChunk
  int32_t u;       // original id of the hub (the parent written to pred)
};

// Slice items of a row [st, st + deg): a row longer than `chunk` (a multiple
// of 128) is cut at multiples of `chunk` elements above the 128-element
// boundary below st, so every item but the row's first and last starts and
// ends on a window boundary of the slice streamer (its windows then carry no
// valid masks and can take the all-hot path); a shorter row is one item.
__host__ __device__ __forceinline__ int slice_items(int64_t st, int32_t deg, int chunk) {
  if (deg <= chunk) return deg > 0 ? 1 : 0;
  return (int)((st + deg - (st & ~int64_t(127)) + chunk - 1) / chunk);
}
__host__ __device__ __forceinline__ CtaItem slice_item(int64_t st, int32_t deg, int chunk, int j, int32_t u) {
  if (deg <= chunk) return CtaItem{st, deg, u};
  const int64_t a0 = st & ~int64_t(127);
  const int64_t lo = a0 + (int64_t)j * chunk > st ? a0 + (int64_t)j * chunk : st;
  const int64_t e = st + deg, hi = a0 + (int64_t)(j + 1) * chunk < e ? a0 + (int64_t)(j + 1) * chunk : e;
  return CtaItem{lo, (int32_t)(hi - lo), u};
}

// A contiguous element range of the small region inside one degree class.
struct alignas(16) DenseTask {
  int64_t p0;   // first col_idx index
  int32_t len;
  int32_t d;    // degree class
};
constexpr int kDenseTask = 4096;  // elements per dense task
constexpr int kDenseNum = 1, kDenseDenom = 2;  // dense when list > region/2
constexpr int64_t kDenseMinElems = (int64_t)1 << 22;  // ... and the small region holds >= 4 M elements

struct Frontier {
  const int32_t* small;    // after a queue-mode level: small/warp-bin queues ...
  const int32_t* warp;
  const CtaItem* cta;      // hub slices (both modes)
  const CtaItem* wslice;   // warp-bin rows as slices (after a bitmap-mode level)
  const int32_t* list;     // ... after a bitmap-mode level: non-hub list + group items
  const GroupItem* items;
  int64_t n_small, n_warp, n_cta, n_items, n_wslice;
  const uint32_t* front;   // frontier bitmap (dense small-region path)
  const DenseTask* dense;
  int64_t n_dense;
  bool dense_warp;         // stream the warp-bin region from the frontier bitmap
  bool front_nc;           // front is read-only for the launch (non-coherent loads)
};

// Degree classes of the small region: internal ids with degree d form the
// contiguous range [T[d+1], T[d]) whose rows are contiguous in col_idx,
// starting at base[d]; T[d] = #vertices with degree >= d.
struct ClassTable {
  int32_t T[kSmallMax + 2];
  int64_t base[kSmallMax + 1];
};

struct LevelArgs {
  const int64_t* row_ptr;   // internal CSR
  const int32_t* col_idx;
  const int32_t* new2old;
  uint32_t* visited;
  uint32_t* prev;           // visited at the last bitmap-mode boundary
  int32_t* pred_int;        // parent (original id) by internal id
  int32_t* level_int;       // level by internal id (-1 unreached)
  const ClassTable* classes;
  unsigned long long* dbg;  // LBFS_COUNT: candidate-write counters (hot, cold)
  int32_t refresh_chunks;   // hub chunks between hot-snapshot refreshes (warp 0)
  int32_t next_level;
  int32_t t_cta, t_warp, t_nz;  // internal-id bin boundaries (local rows)
  // queue-mode winners with id < t_hub emit their rows as slice items
  // (t_warp: hubs and warp-bin rows — the next level streams them with the
  // descriptor in hand, no row_ptr round trip per row; t_cta: hubs only)
  int32_t t_hub;
  int32_t align_items;      // queue-mode winners cut slice items on 128-element window boundaries
  // partitioned run (nparts = 1 << part_log > 1): this rank owns the ids of
  // bitmap words w with w % nparts == part_rank; pred_int/level_int, rows and
  // frontier entries use local row ids, bitmaps and neighbours global ids
  int32_t part_log, part_rank;
  // queue-mode outputs (direct append by the winners)
  Counters* next_cnt;
  int32_t* next_small;
  int32_t* next_warp;
  CtaItem* next_cta;
  int32_t qchunk;           // edges per hub item appended by a queue-mode winner (<= kChunk)
  // heavy bitmap levels (k_expand<kHeavy>): each CTA ORs hot targets blindly
  // into its zeroed shared copy of the hot prefix and leaves it in row
  // blockIdx.x of stage (hot_words words per row); stage_first: the first
  // launch of the level stores the row, later launches OR into it
  uint32_t* stage;
  int32_t stage_first;
  int32_t stage_words;      // row stride of stage (>= the kernel's hot words: the sweep's prefix can be longer)
  int64_t chk_n, chk_nnz;   // sizes for the LBFS_CHECKS debug build's bounds checks
};

struct CompactArgs {
  const int64_t* row_ptr;
  const int32_t* new2old;
  const uint32_t* visited;
  uint32_t* prev;           // visited at the previous level boundary
  int64_t nwords;           // local (owned) words
  int32_t* level_int;
  int32_t next_level;
  int32_t t_cta, t_warp, t_nz;
  Counters* next_cnt;
  int32_t* next_list;
  CtaItem* next_cta;
  GroupItem* next_items;
  CtaItem* next_wslice;
  uint32_t* front;
  int32_t part_log, part_rank;
  uint32_t* fsend;          // partitioned: owned words of the next frontier (all-gather input)
  // heavy levels: parents of the new vertices with internal id < resolve_verts
  // (the hot prefix, discovered by blind ORs) are resolved here: the first
  // neighbour whose level is cur_level (0 = off)
  const int32_t* col_idx;
  const int32_t* first_nbr;  // first (highest-degree) neighbour of each row
  int32_t* pred_int;
  int32_t resolve_verts;
  int32_t cur_level;
};

// Owner / local id of a global internal id (word-cyclic partition).
__host__ __device__ __forceinline__ bool part_owned(int32_t v, int32_t part_log, int32_t part_rank) {
  return ((v >> 5) & ((1 << part_log) - 1)) == part_rank;
}
__host__ __device__ __forceinline__ int32_t part_local(int32_t v, int32_t part_log) {
  return (((v >> 5) >> part_log) << 5) | (v & 31);
}
__host__ __device__ __forceinline__ int64_t part_global(int64_t l, int32_t part_log, int32_t part_rank) {
  return ((((l >> 5) << part_log) | part_rank) << 5) | (l & 31);
}

// Programmatic dependent launch (see LBFS_LAUNCH_PDL): both are no-ops in a
// kernel launched the plain way.
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Heavy levels, a lane's four consecutive elements of a sorted row, all in the
// hot prefix: blind ORs into the CTA's shared copy (shared-window address
// `base`), with runs in one bitmap word merged into a single reduction. The
// shared-atomic pipe bounds the heavy kernels (ncu: ~3.7 wavefronts per
// ATOMS from bank and same-word conflicts), and in hub rows ~45% of the
// elements share a word with their predecessor.
__device__ __forceinline__ void heavy_or_hot4(uint32_t base, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile(
      "{\n\t"
      ".reg .pred p1, p2, p3;\n\t"
      ".reg .u32 ax, ay, az, aw, bx, by, bz, bw;\n\t"
      "shf.l.wrap.b32 bx, 0, 1, %0;\n\t"
      "shf.l.wrap.b32 by, 0, 1, %1;\n\t"
      "shf.l.wrap.b32 bz, 0, 1, %2;\n\t"
      "shf.l.wrap.b32 bw, 0, 1, %3;\n\t"
      "shr.u32 ax, %0, 5;\n\t"
      "shr.u32 ay, %1, 5;\n\t"
      "shr.u32 az, %2, 5;\n\t"
      "shr.u32 aw, %3, 5;\n\t"
      "setp.ne.u32 p1, ax, ay;\n\t"
      "setp.ne.u32 p2, ay, az;\n\t"
      "setp.ne.u32 p3, az, aw;\n\t"
      "@!p1 or.b32 by, by, bx;\n\t"
      "@!p2 or.b32 bz, bz, by;\n\t"
      "@!p3 or.b32 bw, bw, bz;\n\t"
      "mad.lo.u32 ax, ax, 4, %4;\n\t"
      "mad.lo.u32 ay, ay, 4, %4;\n\t"
      "mad.lo.u32 az, az, 4, %4;\n\t"
      "mad.lo.u32 aw, aw, 4, %4;\n\t"
      "@p1 red.shared.or.b32 [ax], bx;\n\t"
      "@p2 red.shared.or.b32 [ay], by;\n\t"
      "@p3 red.shared.or.b32 [az], bz;\n\t"
      "red.shared.or.b32 [aw], bw;\n\t"
      "}" ::"r"(x),
      "r"(y), "r"(z), "r"(w), "r"(base)
      : "memory");
}

// ... one target, valid in every lane, hot or cold: the word index decides
// between the shared copy and visited in L2 (ptxas turns the two predicated
// reductions into short forward branches; no other control flow).
__device__ __forceinline__ void heavy_or_any(uint32_t base, uint32_t hot_words, const uint32_t* visited, uint32_t v) {
  asm volatile(
      "{\n\t"
      ".reg .pred ph;\n\t"
      ".reg .u32 wi, sa, bit;\n\t"
      ".reg .u64 ga;\n\t"
      "shr.u32 wi, %0, 5;\n\t"
      "shf.l.wrap.b32 bit, 0, 1, %0;\n\t"
      "setp.lt.u32 ph, wi, %1;\n\t"
      "mad.lo.u32 sa, wi, 4, %2;\n\t"
      "mad.wide.u32 ga, wi, 4, %3;\n\t"
      "@ph red.shared.or.b32 [sa], bit;\n\t"
      "@!ph red.relaxed.gpu.global.or.b32 [ga], bit;\n\t"
      "}" ::"r"(v),
      "r"(hot_words), "r"(base), "l"(visited)
      : "memory");
}

// ... one target, valid when ok != 0
__device__ __forceinline__ void heavy_or_ok(uint32_t base, uint32_t hot_words, const uint32_t* visited, uint32_t v,
                                            uint32_t ok) {
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
      "mad.lo.u32 sa, wi, 4, %3;\n\t"
      "mad.wide.u32 ga, wi, 4, %4;\n\t"
      "@ph red.shared.or.b32 [sa], bit;\n\t"
      "@pc red.relaxed.gpu.global.or.b32 [ga], bit;\n\t"
      "}" ::"r"(v),
      "r"(ok), "r"(hot_words), "r"(base), "l"(visited)
      : "memory");
}

constexpr int64_t kLoopCap = 1 << 16;  // levels per cluster-kernel launch

// Small-frontier levels on one thread-block cluster (cluster.cu).
constexpr int kClusterThreads = 512;
constexpr unsigned long long kClusterExitEdges = 1ull << 16;  // default LBFS_CLUSTER_EDGES
constexpr unsigned long long kClusterExitHubEdges = 1ull << 14;  // default LBFS_CLUSTER_HUB_EDGES
// A frontier stays on the cluster while it is thin: at most exit_edges edges
// (a lattice level: thousands of vertices of degree <= 4), and at most
// exit_hub_edges when its rows are long (average degree > 32: an R-MAT level
// of hubs, which 16 SMs stream slowly and the full grid takes in one step).
__host__ __device__ __forceinline__ bool cluster_takes(unsigned long long verts, unsigned long long edges,
                                                       unsigned long long exit_edges,
                                                       unsigned long long exit_hub_edges) {
  return edges <= exit_edges && !(edges > exit_hub_edges && edges > 32ull * verts);
}
constexpr int kMaxCluster = 16;
constexpr int kClusterStage = 128;  // winners staged per target CTA before the push
// A frontier entry of the cluster's small queues: the vertex (internal id)
// and its parent (original id); its level / parent records are written when
// it is expanded (early in the next level, off the level's critical chain).
struct alignas(8) QEntry {
  int32_t v;
  int32_t par;
};
struct ClusterArgs {
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const int32_t* new2old;
  const int32_t* old2new;
  const ClassTable* classes;
  int32_t t_cta, t_warp, t_nz;
  int32_t root_orig;        // >= 0: the first level of a BFS (visited = {root}: no bitmap load)
  uint32_t* visited;
  uint32_t* prev;
  int32_t* pred_int;
  int32_t* level_int;
  int64_t nwords;
  int64_t slice_words;      // DSMEM mode: bitmap words per CTA (multiple of 8)
  int32_t qs;               // entries per shared-memory small queue
  int32_t mail_cap;         // DSMEM mode: candidates per sender in a CTA's mailbox area (0: remote claims)
  int32_t qchunk;           // edges per exit slice item (at most)
  int32_t exit_warps;       // warps of the full-GPU queue-mode grid (0: fixed qchunk items)
  int64_t cap;              // spill / big-list capacity per buffer (>= exit_edges)
  // frontier of level L0 (counters in ring[L0 % 3]): the host's queue format,
  // or a bitmap level's list (in_small) + warp slices (in_items2) + hub slices
  const int32_t* in_small;
  const int32_t* in_warp;
  const CtaItem* in_items;
  const CtaItem* in_items2;
  int32_t in_bitmap;        // 1: the list format (counts bin[kBinSmall / kBinWSlice / kBinCta])
  Counters* ring;
  int64_t L0, max_levels;
  unsigned long long exit_edges;  // leave when a frontier has more edges
  unsigned long long exit_hub_edges;  // ... or more than this many with an average degree above 32 (hub rows)
  unsigned long long bitmap_min_edges;  // the host's next level is bitmap mode from this many edges
  int32_t* out_small[2];    // exit frontier (queue format) by level parity
  CtaItem* out_cta[2];
  QEntry* spill_small;      // [kMaxCluster][2][cap]
  CtaItem* big;             // [3][cap] cluster-wide lists of degree >= 32 rows
  unsigned long long* big_cnt;  // [3]
  lbfs_layer* layers;       // layers[L - L0] (mapped host memory)
  Counters* mail;
  unsigned long long* seq;
  unsigned long long seq_value;
  int32_t dbg;               // LBFS_CLUSTER_DBG experiments (wrong results): 1 no prefetch, 2 no layers, 4 no level/pred stores
  int64_t prof_level;        // LBFS_CLUSTER_PROF_LEVEL: per-warp timeline of this level (CTA rank 0)
  unsigned long long* prof;  // LBFS_CLUSTER_PROF: [0] start [1] slices loaded [2] exit; 8 + 4 L: level stamps
};
template <bool DSM>
__global__ void k_cluster_levels(const __grid_constant__ ClusterArgs p);
size_t cluster_static_smem();

// Heavy-level sweep of the big-row region (sweep.cu).
constexpr int kSweepWindow = 128;   // col_idx elements per window / side entry
#ifndef LBFS_SWEEP_CONSUMERS
#define LBFS_SWEEP_CONSUMERS 16
#endif
constexpr int kSweepConsumers = LBFS_SWEEP_CONSUMERS;  // consumer warps; one CTA per SM
constexpr int kSweepProducers = 4;   // producer warps (each a latency-bound side -> frontier -> copy chain)
#ifndef LBFS_SWEEP_WORKERS
#define LBFS_SWEEP_WORKERS 0
#endif
// (experiment, off: with 4 worker warps S24 measured 385 vs 402 GTEPS — the
// extra warps slow the ring's consumers by more than the saved launch)
// worker warps: the dense small region's tasks, streamed next to the ring
constexpr int kSweepWorkers = LBFS_SWEEP_WORKERS;
constexpr int kSweepThreads = 32 * (kSweepConsumers + kSweepProducers + kSweepWorkers);
#ifndef LBFS_SWEEP_STAGES
#define LBFS_SWEEP_STAGES 4
#endif
constexpr int kSweepStages = LBFS_SWEEP_STAGES;  // ring depth (16 KB chunks)
#ifndef LBFS_SWEEP_MIN_PCT
#define LBFS_SWEEP_MIN_PCT 30
#endif
#ifndef LBFS_BITMAP_DIV
#define LBFS_BITMAP_DIV 16
#endif
constexpr int kBitmapDiv = LBFS_BITMAP_DIV;  // bitmap-mode output when a frontier's edges >= max(2^16, n / this)
constexpr int kHeavyDiv = 32;  // heavy (blind-OR) semantics when a bitmap level's edges >= nnz / this
constexpr int kSweepMinPct = LBFS_SWEEP_MIN_PCT;  // sweep a heavy level when its big-row edges >= this % of e_big
constexpr int kSweepPrefetch = 0;    // L2 prefetch distance (chunks of a CTA)
#ifndef LBFS_SWEEP_CHUNK_WINS
#define LBFS_SWEEP_CHUNK_WINS 32
#endif
constexpr int kSweepChunkWins = LBFS_SWEEP_CHUNK_WINS;  // windows per chunk (<= 32: one producer lane each), a multiple of the consumer warps
static_assert(kSweepChunkWins <= 32 && kSweepChunkWins % kSweepConsumers == 0, "sweep chunk shape");
constexpr int kSweepRingBytes = kSweepStages * kSweepChunkWins * kSweepWindow * 4;
struct SweepArgs {
  const int32_t* col_idx;
  const uint2* side;        // per window: {row of its first element, offsets of rows starting inside}
  int64_t nwin;             // windows of [0, e_big) (side entries)
  int64_t e_big;            // end of the rows of degree >= 32 (ids [0, t_warp))
  int64_t nwin_all;         // windows of [0, e_end): the whole sweep
  int64_t e_end;            // end of the small region (rows of degree 1..31)
  int64_t w_small0;         // first window holding small-region elements (e_big / 128)
  const uint4* svmask;      // valid masks of windows [w_small0, nwin_all) (k_sweep_plan_small)
  const uint32_t* front;    // frontier bitmap of the level (internal ids)
  uint32_t* visited;
  int32_t* pred_int;
  const int32_t* new2old;
  uint32_t* stage;          // per-CTA rows of the hot prefix (see LevelArgs::stage)
  int32_t stage_first;
  int32_t stage_words;      // row stride of stage
  int32_t hot_words;
  int32_t prefetch;         // L2 prefetch distance in chunks of a CTA (0: off)
  int32_t dbg_flags;        // LBFS_SWEEP_DBG (experiments; wrong results): 1 no hot ORs, 2 no cold probes
  // dense small region (rows of degree 1..31, most of them in the frontier):
  // its tasks go to the worker warps (n_dense 0: none)
  const DenseTask* dense;
  int64_t n_dense;
  const ClassTable* classes;
};
// Heavy levels as one window stream over [0, e_nz) (stream.cu).
constexpr int kStreamThreads = 1024;
#ifndef LBFS_STREAM_DEPTH
#define LBFS_STREAM_DEPTH 2
#endif
constexpr int kStreamDepth = LBFS_STREAM_DEPTH;  // windows per group (two groups in flight per warp)
struct StreamArgs {
  const int32_t* col_idx;
  const uint4* wmask;     // valid masks of the big-row windows [0, nwin_big)
  const uint4* svmask;    // ... of the small-row windows [w_small0, nwin)
  int64_t nwin, nwin_big, w_small0;
  uint32_t* visited;
  uint32_t* stage;        // per-CTA rows of the hot prefix (LevelArgs::stage)
  int32_t stage_words;
  int32_t hot_words;
};
__global__ void k_window_masks(const uint2* side, int64_t nwin, int64_t e_big, const uint32_t* front,
                               const uint4* svmask, int64_t w_small0, uint4* wmask);
template <int D>
__global__ void k_stream_heavy(const __grid_constant__ StreamArgs s);

struct BottomUpArgs {
  const int64_t* row_ptr;
  const int32_t* col_idx;
  const int32_t* new2old;
  const uint32_t* front;   // frontier bitmap of the level
  uint32_t* visited;
  int32_t* pred_int;
  int64_t nwords;          // visited words covering [0, t_nz)
  int64_t t_nz;            // rows of degree >= 1 are [0, t_nz)
};
__global__ void k_bottom_up(const BottomUpArgs b);
__global__ void k_front_from_queues(uint32_t* front, const int32_t* qs, int64_t ns, const int32_t* qw, int64_t nw,
                                    const CtaItem* qc, int64_t nc, const int32_t* old2new);
__global__ void k_side_table(const int64_t* rp, int32_t nrows, int64_t nwin, uint2* side);
__global__ void k_sweep(const __grid_constant__ SweepArgs s);
__global__ void k_resolve(const int32_t* level_int, const int32_t* first_nbr, const int64_t* row_ptr,
                          const int32_t* col_idx, const int32_t* new2old, int32_t* pred_int, int64_t n, int32_t lvl);
__global__ void k_small_desc(const ClassTable* classes, int64_t e_big, int64_t e_end, int64_t w0, int64_t nw,
                             uint2* desc);
__global__ void k_sweep_plan_small(const ClassTable* classes, const uint2* desc, const uint32_t* front, int64_t e_end,
                                   int64_t w0, int64_t nw, uint4* svmask);

bool env_flag(const char* name);
__global__ void k_init(uint4* vis4, uint4* prev4, int64_t nwords4, int4* lvl4, int64_t n4,
                       Counters* ring = nullptr);
__global__ void k_seed(LevelArgs a, uint32_t* prev, const int32_t* old2new, int32_t root_orig, Counters* cnt0,
                       uint32_t* fglob, unsigned long long* red);
unsigned clamp_grid(int64_t blocks, int64_t cap);

class BfsEngine {
 public:
  // Builds the internal layout from a device CSR in original ids (not kept).
  // nparts > 1 (a power of two): the partition of rank `rank` only
  // (multi-GPU, partition.cu); run() needs nparts == 1.
  explicit BfsEngine(const Csr& csr, int rank = 0, int nparts = 1);
  ~BfsEngine();
  BfsEngine(const BfsEngine&) = delete;
  BfsEngine& operator=(const BfsEngine&) = delete;

  void ensure_own_outputs();
  // BFS into device buffers d_pred[pad32(n)], d_level[n]; synchronous.
  // direction: 0 top-down, 1 direction-optimising (bottom-up levels)
  void run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t, int direction = 0);
  // BFS with host outputs (parents D2H overlapped with the output pass)
  void run_to_host(int64_t root, int direction, int32_t* h_pred, int32_t* h_level, lbfs_timing* t);
  // levels of the last BFS (original ids) to host memory
  void last_levels_to_host(int32_t* h_level);

  // ---- partitioned BFS, one level step at a time (partition.cu); the
  // collectives between the steps are issued by the caller on `st`
  void part_start(int64_t root, cudaStream_t st, unsigned long long* red);
  void part_expand(cudaStream_t st);
  void part_pack(uint32_t* send, cudaStream_t st);
  void part_merge(const uint32_t* recv, uint32_t* fsend, cudaStream_t st);
  void part_sync(const uint32_t* fgath, cudaStream_t st);
  void part_level_done(const unsigned long long* red_global, lbfs_layer* layer, int* done);
  void part_finish(int32_t* d_pred, int32_t* d_level, cudaStream_t st);
  // words per peer of the coming level's all-to-all / per rank of its all-gather
  void part_plan(int64_t* a2a_words, int64_t* gather_words) const;
  int nparts() const { return nparts_; }
  int part_rank() const { return part_rank_; }
  int64_t nwords() const { return nwords_; }
  int64_t n_local() const { return n_loc_; }
  int64_t nnz_local() const { return nnz_loc_; }
  unsigned long long resolve_scanned() const;
  // validate_tree (validate.py:50-155) on a device parent array in original
  // ids: out[0..4] passed flags, out[5..9] details (-1 when passed)
  void validate_tree(int64_t root, const int32_t* d_pred, int64_t out[10]);
  int64_t n() const { return n_; }
  int64_t nnz() const { return nnz_; }
  int64_t npad() const { return npad_; }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  int32_t* own_pred() const { return own_pred_; }
  int32_t* own_level() const { return own_level_; }
  const std::vector<lbfs_layer>& layers() const { return layers_; }

  std::mutex mu;

 private:
  void build_layout(const Csr& csr);
  void launch_expand(int mode, int pi, unsigned grid, const LevelArgs& a, const Frontier& f, cudaStream_t st,
                     bool pdl = false);
  LevelArgs level_args() const;
  // frontier of level L (queue slot cur, counters c) -> launches; returns the grid
  // mode: 0 bitmap, 1 queue, 3 heavy bitmap (blind hot ORs, see LevelArgs::stage)
  unsigned bottom_up_level(const Counters& c, bool prev_bitmap, int cur, cudaStream_t st);
  unsigned expand_level(LevelArgs& a, const Counters& c, int mode, bool prev_bitmap, int cur, int64_t L,
                        cudaStream_t st);
  void compact_level(int cur, int64_t L, uint32_t* fsend, cudaStream_t st, bool heavy = false, bool pdl = false);
  void merge_hot(cudaStream_t st);
  void launch_resolve(int64_t lvl, cudaStream_t st);
  void flush_resolve(cudaStream_t st);
  void read_env();
  void finalize(int32_t* d_pred, int32_t* d_level, cudaStream_t st);
  void levels_out(int32_t* d_level, cudaStream_t st);
  static constexpr int kOutChunks = 8;
  int32_t* host_pred_ = nullptr;     // run_to_host: parents' host destination
  cudaStream_t out_st_ = nullptr;    // D2H of the outputs
  cudaEvent_t ev_out_[kOutChunks] = {};
  void setup_cluster(int optin);
  void launch_cluster(int64_t L, int cur, bool prev_bitmap, cudaStream_t st, int32_t root_orig);
  bool split_any_ = false;

  int device_ = 0, sm_count_ = 0;
  int64_t n_ = 0, nnz_ = 0, nwords_ = 0, npad_ = 0;  // global: vertices, entries, bitmap words, pad32(n)
  int nparts_ = 1, part_rank_ = 0, part_log_ = 0;
  int64_t n_loc_ = 0, nwl_ = 0, nnz_loc_ = 0;       // this rank: rows, owned words, entries
  int32_t* new2old_loc_ = nullptr;                  // local row -> original id (== new2old_ if nparts 1)
  // partitioned state
  uint32_t* fglob_ = nullptr;                       // replicated frontier bitmap of the current level
  unsigned long long* resolve_cnt_ = nullptr;       // adjacency entries read by parent resolution
  int64_t part_L_ = 0;
  int part_cur_ = 0;
  bool part_prev_bitmap_ = false;
  cudaStream_t part_st_ = nullptr;
  unsigned long long part_in_ = 0, part_edges_ = 0;  // global counts of the current frontier
  unsigned long long* h_red_ = nullptr;              // pinned: global (discovered, edges)
  unsigned long long* red_dev_ = nullptr;            // summed counts of the gathered slices
  int64_t* row_ptr_ = nullptr;   // internal CSR
  int32_t* col_idx_ = nullptr;
  int32_t* new2old_ = nullptr;
  int32_t* old2new_ = nullptr;
  int32_t t_cta_ = 0, t_warp_ = 0, t_nz_ = 0;
  ClassTable* classes_ = nullptr;
  unsigned long long* dbg_ = nullptr;
  uint32_t* visited_ = nullptr;
  uint32_t* prev_ = nullptr;
  int32_t* pred_int_ = nullptr;
  int32_t* level_int_ = nullptr;
  uint32_t* front_ = nullptr;
  DenseTask* dense_tasks_ = nullptr;
  int64_t n_dense_tasks_ = 0;
  bool dense_off_ = false;
  int dense_pct_ = 100 * kDenseNum / kDenseDenom;
  int64_t dense_min_elems_ = kDenseMinElems;
  bool dense_warp_ = false;
  int32_t* q_small_[2] = {nullptr, nullptr};
  int32_t* q_warp_[2] = {nullptr, nullptr};
  CtaItem* q_cta_[2] = {nullptr, nullptr};
  GroupItem* q_items_[2] = {nullptr, nullptr};
  CtaItem* q_wslice_[2] = {nullptr, nullptr};
  int64_t cap_cta_ = 0, cap_items_ = 0;
  Counters* cnt_ = nullptr;
  Counters* h_cnt_ = nullptr;
  // per-level mailbox in mapped pinned memory: the cluster kernel (or
  // k_publish) copies a frontier's counters here and bumps the sequence word;
  // the host spins on it
  Counters* h_mail_ = nullptr;
  unsigned long long* h_seq_ = nullptr;
  unsigned long long seq_ = 0;
  void publish_and_wait(int slot, int zero_slot, cudaStream_t st);
  void wait_mail(unsigned long long want, cudaStream_t st);
  lbfs_layer* h_loop_layers_ = nullptr;  // mapped: the cluster kernel's per-level layers of the current run
  int32_t* own_pred_ = nullptr;
  int32_t* own_level_ = nullptr;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_[7] = {};
  cudaEvent_t ev_gap_ = nullptr;
  static constexpr int kClEvents = 16;
  cudaEvent_t ev_cl_[2 * kClEvents] = {};  // cluster segments of one BFS (timing)
  int n_cl_ev_ = 0;
  std::vector<lbfs_layer> layers_;
  int expand_grid_ = 0;
  // cluster level loop (cluster.cu)
  int cl_size_ = 0;               // CTAs per cluster (0: unavailable)
  bool cl_dsm_ = false;           // visited bitmap in distributed shared memory
  bool cl_no_dsm_ = false, cl_off_ = false;
  bool qgrid_old_ = false;
  bool compact_big_ = false;
  bool lean_events_ = false;
  int64_t resolve_deferred_ = -1;
  bool align_items_ = false;
  bool sweep_workers_ = true;
  bool cl_dsm_always_ = false;
  bool exit_fair_ = true;
  bool fuse_queues_ = true;
  bool publish_after_heavy_ = true;
  bool resolve_inline_ = false, resolve_clamp_ = false;
  bool warp_items_ = true;
  int64_t cl_slice_words_ = 0;
  int32_t cl_qs_ = 0;
  int32_t cl_mail_cap_ = 0;
  bool cl_no_mail_ = false;
  int cl_mail_cap_env_ = 0;
  int cl_smem_ = 0;
  int64_t cl_cap_ = 0;
  unsigned long long cl_exit_edges_ = kClusterExitEdges;
  unsigned long long cl_exit_hub_edges_ = kClusterExitHubEdges;
  QEntry* cl_spill_ = nullptr;
  CtaItem* cl_big_ = nullptr;
  unsigned long long* cl_big_cnt_ = nullptr;
  bool cl_prof_ = false;
  int cl_dbg_ = 0;
  int cl_force_size_ = 0;
  long long cl_prof_level_ = -1;
  unsigned long long* cl_prof_buf_ = nullptr;
  int32_t hot_words_ = 0;  // visited words mirrored in shared memory
  int32_t sweep_hot_words_ = 0;  // the sweep's (longer) hot prefix
  int32_t stream_hot_words_ = 0; // k_stream_heavy's hot prefix (longest: no ring next to it)
  int32_t stage_words_ = 0;      // stage row stride (>= every kernel's hot prefix)
  int32_t merge_words_ = 0;      // hot words written to the stage rows by this level's kernels
  uint4* wmask_ = nullptr;       // k_stream_heavy: valid masks of the big-row windows
  bool stream_on_ = false;       // LBFS_STREAM=1: heavy levels as one full-CSR window stream (experiment)
  bool sweep_after_queue_ = false;  // LBFS_SWEEP_AFTER_QUEUE=1: sweep heavy levels that follow a queue level
  uint32_t* stage_ = nullptr;    // heavy levels: expand_grid_ rows of hot_words_ words
  uint2* side_ = nullptr;        // sweep side entries (nparts 1)
  int32_t* first_nbr_ = nullptr; // first neighbour of each row (heavy-level parent resolution)
  uint4* svmask_ = nullptr;      // sweep: per-level valid masks of the small-region windows
  uint2* sdesc_ = nullptr;       // sweep: small-region window descriptors (k_small_desc)
  int64_t e_nz_ = 0, n_win_all_ = 0, w_small0_ = 0;
  int64_t n_side_win_ = 0, e_big_ = 0;
  bool sweep_off_ = false;       // LBFS_NO_SWEEP=1: heavy levels use the slice lists
  bool sweep_used_ = false;      // the last expand_level swept the big-row region
  bool sweep_fits_ = false;      // k_sweep's ring + hot prefix fit in shared memory
  cudaStream_t res_st_ = nullptr;  // heavy-level parent resolution (k_resolve), joined before k_finalize
  cudaEvent_t ev_resolve_ = nullptr, ev_side_done_ = nullptr;
  bool side_pending_ = false;
  bool sweep_small_ = false;     // LBFS_SWEEP_SMALL=1: sweep the small region as well (slower today)
  int heavy_div_ = kHeavyDiv;    // heavy when a bitmap level's edges >= nnz / heavy_div_ (0: off)
  int heavy_vis_pct_ = 0;        // ... and the visited edge mass <= this % of the frontier's (0: no limit)
  int dyn_smem_ = 0;
  bool trace_ = false;  // LBFS_TRACE=1: per-level table on stderr
  int sweep_min_pct_ = kSweepMinPct;
  int bu_alpha_ = 14, bu_beta_ = 24;
  int bitmap_div_ = kBitmapDiv;
  int64_t bitmap_floor_ = (int64_t)1 << 16;
  int refresh_chunks_ = kRefreshChunks;
  int qchunk_ = kQChunkDefault;
  bool part_heavy_ = false;      // this partition level runs with heavy (blind-OR) semantics
  uint32_t* snap_[2] = {nullptr, nullptr};  // F_L snapshots for k_part_resolve (heavy levels)
  cudaEvent_t ev_snap_[2] = {nullptr, nullptr};
  bool snap_used_[2] = {false, false};
  int snap_next_ = 0;
  const uint32_t* part_fgath_ = nullptr;  // the gathered slices of the level (part_sync -> part_level_done)
  // sparse exchange of the current level (partition.cu): S words per peer in
  // the all-to-all, G per rank in the all-gather
  bool part_sparse_ = false;
  int part_sparse_mode_ = 1;  // LBFS_PART_SPARSE: 0 never, 1 when 2 (E_L + 8) <= W, 2 whenever E_L + 8 <= W
  int64_t part_S_ = 0, part_G_ = 0;
  uint32_t* part_send_ = nullptr;  // the level's send slices (own marks -> prev after a sparse level)
  unsigned long long* part_err_ = nullptr;
  void part_choose_format();
  bool part_heavy_off_ = false;  // LBFS_PART_HEAVY=0
  bool count_ = false;
  bool split_ = false;
  cudaEvent_t ev_split_[7] = {};  // LBFS_COUNT=1: count bitmap-mode candidate writes (slow)
};

}  // namespace lbfs

#include "multi.cuh"

struct lbfs_graph {
  lbfs::BfsEngine* eng = nullptr;     // one GPU (or one partition, lbfs_part_*)
  lbfs::MultiGraph* multi = nullptr;  // ngpus > 1: partitions on several devices of this process
};
