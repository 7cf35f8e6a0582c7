/*
 * lbfs.h — C ABI of the B200-native top-down BFS (sm_100a).
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `lanebfs` (arXiv 1604.02844): everything below `run_bfs(g, s, policy)`
 * (reference pkg/src/lanebfs/traversal.py:413-422) and the graph inputs it
 * consumes (graph.py:68-160). Plain pointers and sizes only; no torch types.
 *
 * Conventions
 *   - Return 0 on success or a negative LBFS_E* code. The message of the last
 *     failure on the calling thread is in lbfs_last_error().
 *   - Vertex ids are int32 (the reference caps SCALE at 30 so ids stay below
 *     the sentinel, graph.py:11-13); CSR offsets are int64 (graph.py:156).
 *   - Host output buffers are caller-owned. Device state is library-owned.
 *   - Calls on one graph handle are serialised by a mutex inside the library
 *     (the reference never overlaps BFS calls).
 */
#ifndef LBFS_H
#define LBFS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBFS_OK 0
#define LBFS_EINVAL (-1) /* bad argument: the Python layer raises AssertionError */
#define LBFS_ECUDA (-2)  /* CUDA runtime / launch failure */
#define LBFS_ENCCL (-3)  /* collective failure (multi-GPU) */
#define LBFS_ENOMEM (-4) /* device or pinned-host allocation failed */

/* Unreached-predecessor value; reference traversal.py:22 (SENTINEL). */
#define LBFS_SENTINEL 0x7FFFFFFF

typedef struct lbfs_graph lbfs_graph; /* device-resident BFS graph        */
typedef struct lbfs_csr lbfs_csr;     /* device-resident CSR (original ids) */

/* One BFS layer; reference LayerStats, traversal.py:66-70. */
typedef struct lbfs_layer {
  int64_t input;      /* frontier vertices entering the layer       */
  int64_t edges;      /* adjacency entries examined (sum of degree)  */
  int64_t discovered; /* vertices first reached in this layer        */
} lbfs_layer;

/* Device-side timing of one BFS. bfs_ms and finalize_ms come from CUDA events
 * on the BFS stream. No event is recorded between the kernels of a BFS (an
 * event there serialises the stream and ends a chain of programmatic
 * dependent launches): cluster_ms is the device time the cluster kernel
 * measured inside its launches, expand_ms the rest of the level loop (init,
 * full-GPU level kernels, launch latency and host round trips), init_ms 0.
 * LBFS_FULL_EVENTS=1 brackets init, every full-GPU level and every cluster
 * launch with events instead (slower; the meanings in the comments below). */
typedef struct lbfs_timing {
  double bfs_ms;           /* init kernel start -> end of the output pass    */
  double init_ms;          /* K4 init (pred/level fill, bitmap clear, seed)  */
  double expand_ms;        /* full-GPU levels: expansion + merge + compaction kernels (summed) */
  double cluster_ms;       /* small-frontier levels on the cluster (summed)  */
  double finalize_ms;      /* output pass (parents / levels in original ids) */
  double d2h_ms;           /* host-output variant: output copy to host       */
  int64_t levels;          /* number of layers (== n_layers)                 */
  int64_t kernel_launches; /* kernels this BFS launched                      */
  int64_t edges;           /* traversed_edge_count (sum of layer edges)      */
  int64_t reached;         /* vertices with a level (sum of layer inputs)    */
} lbfs_timing;

typedef struct lbfs_device_info {
  int device;
  int sm_count;
  int cc_major;
  int cc_minor;
  int64_t l2_bytes;
  int64_t hbm_bytes;
  int64_t smem_per_block_optin;
  char name[256];
} lbfs_device_info;

/* ---- library ---------------------------------------------------------- */

/* Thread-local message of the last failing call ("" if none). */
const char* lbfs_last_error(void);
/* Make `device` the calling thread's device for subsequent construction
 * calls (one process per GPU: the local rank's device). */
int lbfs_set_device(int device);
/* Properties of CUDA device `device`. */
int lbfs_device_info_get(int device, lbfs_device_info* out);
/* Number of kernel launches this process has issued through the library. */
int64_t lbfs_kernel_launch_count(void);
/* Page-locked host memory for BFS outputs (D2H at full PCIe rate); the
 * Python layer pools these buffers behind the numpy arrays it returns. */
int lbfs_host_alloc(int64_t bytes, void** out);
void lbfs_host_free(void* p);

/* ---- graph construction (reference graph.py) -------------------------- */

/* R-MAT endpoint pairs, bit-exact with the reference generate_rmat
 * (graph.py:68-85): numpy Generator(PCG64).random() draws in the same order.
 * pcg = {state_hi, state_lo, inc_hi, inc_lo} of default_rng(seed)'s PCG64.
 * Host outputs src/dst of length m = 2^scale * edgefactor. */
int lbfs_rmat_edges(int scale, int64_t m, double ab, double a_norm, double c_norm,
                    const uint64_t pcg[4], uint32_t* src_out, uint32_t* dst_out);

/* Seeded vertex permutation (Feistel bijection on [0,n))
 * applied in place to both endpoint arrays (host). */
int lbfs_permute_edges(int64_t n, uint64_t seed, uint32_t* src, uint32_t* dst, int64_t m);

/* CSR from host endpoint arrays; reference build_csr (graph.py:139-160):
 * symmetrize inserts reverse pairs; dedup sorts each row, drops duplicates
 * and self-loops; without dedup rows keep stable source order. */
int lbfs_csr_build(int64_t n, const uint32_t* src, const uint32_t* dst, int64_t m,
                   int symmetrize, int dedup, lbfs_csr** out);
/* Whole pipeline on the device: generate_rmat -> (optional) permutation ->
 * build_csr(symmetrize=True, dedup=True). No host copy of the edge list. */
int lbfs_csr_build_rmat(int scale, int edgefactor, double ab, double a_norm, double c_norm,
                        const uint64_t pcg[4], int permute, uint64_t perm_seed, lbfs_csr** out);
/* 2D 4-neighbour lattice rows x cols (vertex r*cols+c, edges right and down,
 * no wrap) -> (optional) permutation -> build_csr on the device. */
int lbfs_csr_build_lattice(int64_t rows, int64_t cols, int permute, uint64_t perm_seed,
                           lbfs_csr** out);
int lbfs_csr_info(const lbfs_csr* csr, int64_t* n, int64_t* nnz);
/* Copy the CSR to host arrays: row_ptr[n+1] (int64), col_idx[nnz] (int32). */
int lbfs_csr_download(const lbfs_csr* csr, int64_t* row_ptr, int32_t* col_idx);
void lbfs_csr_destroy(lbfs_csr* csr);

/* ---- BFS graph handle (replaces CsrGraph as seen by run_bfs) ---------- */

/* Copy a host CSR (colstarts int64[n+1], rows int32[nnz]; graph.py:96-136) to
 * the device and build the traversal layout. ngpus == 1: one GPU
 * (the current device). ngpus > 1 (a power of two): the graph is
 * 1D-partitioned over devices 0..ngpus-1 of this process, one partition per
 * device, with one library-owned NCCL communicator per device
 * (ncclCommInitAll; libnccl.so.2 is loaded at run time) — lbfs_bfs then runs
 * the partitioned level loop from the calling thread (ncclGroupStart/End per
 * collective) and returns the same outputs. */
int lbfs_graph_create(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                      int ngpus, lbfs_graph** out);
/* Same, from a device CSR (no host round trip). The csr may be destroyed
 * afterwards. */
int lbfs_graph_create_from_csr(const lbfs_csr* csr, int ngpus, lbfs_graph** out);
/* The partitioned path with explicit devices (devices[p] holds partition p;
 * NULL = 0..ngpus-1), also for ngpus == 1 (a one-rank communicator: the
 * partitioned code path on a single GPU). Not for validation (unpartitioned
 * handles only). */
int lbfs_graph_create_partitioned(const lbfs_csr* csr, int ngpus, const int* devices, lbfs_graph** out);
/* Devices a graph handle spans (1 unless partitioned). */
int lbfs_graph_gpus(const lbfs_graph* g, int* ngpus);
void lbfs_graph_destroy(lbfs_graph* g);
int lbfs_graph_info(const lbfs_graph* g, int64_t* n, int64_t* nnz);

/* Traversal direction of one BFS call: LBFS_DIR_TOP_DOWN (the paper's
 * algorithm, the benchmarked path) or LBFS_DIR_OPTIMIZING (bottom-up levels
 * while the frontier is large, Beamer's alpha = 14 / beta = 24 rule; SURVEY
 * §8(f) rank 4). Levels, visited set and layers are identical in both;
 * parents may differ (any neighbour one level up). No reference counterpart:
 * the reference is top-down only. */
#define LBFS_DIR_TOP_DOWN 0
#define LBFS_DIR_OPTIMIZING 1

/* BFS from root; synchronous. Replaces run_bfs/bfs_* (traversal.py:80-422).
 * pred_out must hold pad32(n) int32 entries (PredecessorArray storage,
 * traversal.py:42-46): parent id, root -> root, unreached and padding ->
 * LBFS_SENTINEL. level_out holds n int32 (-1 = unreached). Either output may
 * be NULL (a NULL level_out skips the level copy; lbfs_graph_last_levels
 * fetches them later). All layers are returned under the handle's lock:
 * layers_out receives min(layers_cap, count) of them and *n_layers the count;
 * with too small a buffer call lbfs_graph_last_layers before the next BFS.
 * t_out may be NULL. */
int lbfs_bfs(lbfs_graph* g, int64_t root, int direction, int32_t* pred_out, int32_t* level_out,
             lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers, lbfs_timing* t_out);
/* Same, writing into DEVICE buffers (e.g. torch CUDA tensors) on the graph's
 * device; no host copy inside. d_level may be NULL. */
int lbfs_bfs_device(lbfs_graph* g, int64_t root, int direction, int32_t* d_pred, int32_t* d_level,
                    lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers,
                    lbfs_timing* t_out);
/* Layers of the most recent BFS on this handle (locked). */
int lbfs_graph_last_layers(lbfs_graph* g, lbfs_layer* out, int64_t cap, int64_t* n_layers);
/* Levels (n int32, -1 = unreached, original ids) of the most recent BFS on
 * this handle, to host memory; valid until the next BFS on the handle. */
int lbfs_graph_last_levels(lbfs_graph* g, int32_t* level_out);

/* ---- tree validation (replaces validate_tree, validate.py:50-155) ------
 * The reference's five checks on a parent array in original ids (n int32;
 * SENTINEL = unreached), with its report semantics: report[0..4] = passed
 * flags of root_self_parent, reachability_closure, tree_edge_existence,
 * level_consistency, cycle_freedom; report[5..9] = the first offender of
 * each (the reference's details), -1 when passed. Unpartitioned handles. */
int lbfs_validate_tree(lbfs_graph* g, int64_t root, const int32_t* pred, int64_t report[10]);
int lbfs_validate_tree_device(lbfs_graph* g, int64_t root, const int32_t* d_pred, int64_t report[10]);

/* ---- partitioned BFS (multi-GPU) --------------------------
 * One process per GPU; rank g of P (a power of two) owns the internal ids of
 * bitmap words w with w % P == g and their rows. The level loop
 * (traversal.py:90/152/366 made level-synchronous across ranks) is driven by
 * the caller, who runs the three collectives between the steps on the same
 * stream (paper_1604_02844_b200/distributed.py does this over
 * torch.distributed/NCCL). Per level, with W = nwords / P:
 *   lbfs_part_expand                      owned frontier -> visited / marks
 *   lbfs_part_pack(send[P*W])             marks by owner       -> all_to_all(send, recv)
 *   lbfs_part_merge(recv[P*W], fsend[W+4]) remote discoveries + parents, next
 *                                         frontier: W owned words + this
 *                                         rank's counts (2 x u64) -> all_gather(fsend, fgath[P*(W+4)])
 *   lbfs_part_sync(fgath)                 replicated frontier / visited,
 *                                         counts summed on the device
 *   lbfs_part_level_done(NULL)            layer + termination (host sync)
 * lbfs_part_start(root, red) is followed by all_reduce_sum(red) and one
 * lbfs_part_level_done(red) (which emits no layer). Buffers are device pointers
 * on the partition's device; `stream` is the caller's cudaStream_t, used as
 * given (NULL = the legacy default stream), so the steps are ordered with the
 * collectives the caller issues on the same stream. */
int lbfs_part_create(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz, int rank,
                     int nparts, lbfs_graph** out);
int lbfs_part_create_from_csr(const lbfs_csr* csr, int rank, int nparts, lbfs_graph** out);
int lbfs_part_info(const lbfs_graph* g, int* rank, int* nparts, int64_t* nwords, int64_t* n_local,
                   int64_t* nnz_local);
int lbfs_part_start(lbfs_graph* g, int64_t root, uint64_t* red, void* stream);
int lbfs_part_expand(lbfs_graph* g, void* stream);
int lbfs_part_pack(lbfs_graph* g, uint32_t* send, void* stream);
int lbfs_part_merge(lbfs_graph* g, const uint32_t* recv, uint32_t* fsend, void* stream);
int lbfs_part_sync(lbfs_graph* g, const uint32_t* fgath, void* stream);
/* red_global: the summed start counts after lbfs_part_start; NULL after a level */
int lbfs_part_level_done(lbfs_graph* g, const uint64_t* red_global, lbfs_layer* layer, int* done);
/* Owned vertices' pred (pad32(n)) / level (n) in original ids; every other
 * entry is LBFS_SENTINEL / -1, so the ranks' outputs combine by min / max. */
int lbfs_part_finish(lbfs_graph* g, int32_t* d_pred, int32_t* d_level, void* stream);
/* The coming level's slice sizes, valid after lbfs_part_level_done: words
 * per peer of the all-to-all (W for bitmaps, or a sparse id list) and per
 * rank of the all-gather (W + 4, or a list). Identical on every rank (they
 * follow from the level's global frontier edges E_L): levels with
 * 2 (E_L + 8) <= W exchange [count, ids...] lists (SURVEY §8e sparse
 * exchange). Buffers stay sized for the dense case. */
int lbfs_part_plan(lbfs_graph* g, int64_t* a2a_words, int64_t* gather_words);
/* Adjacency entries read by parent resolution since lbfs_part_start. */
int lbfs_part_resolve_count(lbfs_graph* g, int64_t* out);

/* The same level loop run by the library (one host thread, no per-step
 * calls from the caller) over a library-owned NCCL communicator, for one
 * partition per process (torchrun-style jobs):
 *   rank 0: lbfs_nccl_unique_id(id); the caller broadcasts the 128 bytes
 *   every rank: lbfs_part_attach_nccl(part, id, nparts, rank)   (collective)
 *   every rank: lbfs_part_bfs(part, root, ...)                  (collective)
 * lbfs_part_bfs writes pred (pad32(n)) / level (n, may be NULL) on the
 * partition's device: with gather != 0 the full arrays on every rank (min /
 * max all-reduce), else only the owned entries (SENTINEL / -1 elsewhere).
 * Synchronous; layers and timing as lbfs_bfs_device (t->bfs_ms is this
 * rank's CUDA-event time). After attaching, lbfs_bfs / lbfs_bfs_device on the
 * handle run it with gather = 1. */
int lbfs_nccl_unique_id(uint8_t id[128]);
int lbfs_part_attach_nccl(lbfs_graph* part, const uint8_t id[128], int nranks, int rank);
int lbfs_part_bfs(lbfs_graph* part, int64_t root, int32_t* d_pred, int32_t* d_level, int gather,
                  lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers, lbfs_timing* t_out);

#ifdef __cplusplus
}
#endif

#endif /* LBFS_H */
