// Tree validation on the device: the five checks of the reference's
// validate_tree (validate.py:50-155) over a parent array in original ids,
// with the reference's report semantics (first offender per check).
//
//   1 root_self_parent      p[s] == s                          (details: s)
//   2 reachability_closure  reached v: 0 <= p[v] < n, p[p[v]] reached
//                                                   (details: smallest v)
//   3 tree_edge_existence   (p[v], v) in adj(p[v]) for reached v != s
//                           (details: smallest bad child of the smallest
//                            parent with one, validate.py:96-106)
//   4 level_consistency     no chase from a reached v runs into a cycle or
//                           off the reached set     (details: smallest v)
//   5 cycle_freedom         every chase ends at the root (details: smallest v)
//
// The memoised parent chases (validate.py:108-141) become pointer jumping:
// J[v] starts at p[v] or a terminal code (root, self-parented pseudo-root,
// chase breaks here = parent out of range or unreached), and ceil(log2 n)+2 in-place
// doubling rounds resolve every chase of length <= n; anything still
// pointing at a vertex is on (or leads into) a cycle. Edge membership uses
// the engine's internal CSR (rows sorted): a binary search of old2new[v] in
// the row of old2new[p[v]].
#include "bfs_engine.cuh"

namespace lbfs {

namespace {
// Terminals of a chase. kTermBreaksHere: this vertex's own parent is out of
// range or unreached — the reference's chase stops here without marking the
// vertex itself (validate.py:122-124: it is never appended to the path), so
// it fails only cycle_freedom, while every vertex whose chase reaches it is
// BROKEN.
constexpr int32_t kTermOk = -1, kTermPseudo = -2, kTermBroken = -3, kTermBreaksHere = -4;

__device__ __forceinline__ void amin(unsigned long long* p, unsigned long long v) { atomicMin(p, v); }

// keys: check slot k holds the smallest failing key (all ones = passed)
__global__ void k_val_init(const int32_t* __restrict__ pred, int64_t n, int32_t root, int32_t* __restrict__ J,
                           unsigned long long* __restrict__ keys) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pred[v];
    int32_t j;
    if (v == root) {
      j = kTermOk;  // a chase reaching s ends there whatever p[s] is (validate.py:114)
    } else if (p == kSentinel || p < 0 || p >= n) {
      j = kTermBreaksHere;  // unreached, or a parent out of range
    } else if (p == v) {
      j = kTermPseudo;
    } else {
      j = p;
    }
    J[v] = j;
    if (p != kSentinel && (p < 0 || p >= n || pred[p] == kSentinel)) amin(&keys[1], (unsigned long long)v);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && pred[root] != root) amin(&keys[0], (unsigned long long)root);
}

// tree edges: thread per reached non-root vertex, binary search in the
// parent's row (internal ids)
__global__ void k_val_edges(const int32_t* __restrict__ pred, int64_t n, int32_t root,
                            const int64_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                            const int32_t* __restrict__ old2new, unsigned long long* __restrict__ keys) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = pred[v];
    if (p == kSentinel || v == root) continue;
    bool ok = false;
    if (p >= 0 && p < n) {
      const int32_t iu = __ldg(old2new + p), iv = __ldg(old2new + v);
      int64_t lo = __ldg(row_ptr + iu), hi = __ldg(row_ptr + iu + 1);
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const int32_t x = __ldg(col_idx + mid);
        if (x < iv) lo = mid + 1; else hi = mid;
      }
      ok = lo < __ldg(row_ptr + iu + 1) && __ldg(col_idx + lo) == iv;
    }
    // order of the reference's loop: parents ascending (as ints), then children
    if (!ok) amin(&keys[2], ((unsigned long long)((int64_t)p + 0x80000000LL) << 32) | (unsigned long long)v);
  }
}

__global__ void k_val_jump(int32_t* __restrict__ J, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t j = J[v];
    if (j >= 0) {
      const int32_t t = J[j];
      J[v] = t == kTermBreaksHere ? kTermBroken : t;
    }
  }
}

__global__ void k_val_status(const int32_t* __restrict__ pred, const int32_t* __restrict__ J, int64_t n, int32_t root,
                             unsigned long long* __restrict__ keys) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    if (pred[v] == kSentinel || v == root) continue;
    const int32_t j = J[v];
    const bool cycle = j >= 0, broken = j == kTermBroken;
    if (cycle || broken) amin(&keys[3], (unsigned long long)v);
    if (j != kTermOk) amin(&keys[4], (unsigned long long)v);
  }
}
}  // namespace

// pred: device int32[n] (original ids). out[0..4] = passed flags,
// out[5..9] = details (-1 when passed).
void BfsEngine::validate_tree(int64_t root, const int32_t* pred, int64_t out[10]) {
  if (nparts_ != 1) throw_inval("validation needs an unpartitioned graph");
  if (root < 0 || root >= n_) throw_inval("root out of range");
  cudaStream_t st = stream_;
  int32_t* J = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_, 1));
  unsigned long long* keys = dev_alloc<unsigned long long>(5);
  try {
    LBFS_CUDA(cudaMemsetAsync(keys, 0xFF, 5 * sizeof(unsigned long long), st));
    const unsigned grid = clamp_grid((n_ + 255) / 256, (int64_t)sm_count_ * 16);
    LBFS_LAUNCH(k_val_init, grid, 256, 0, st, pred, n_, (int32_t)root, J, keys);
    LBFS_LAUNCH(k_val_edges, grid, 256, 0, st, pred, n_, (int32_t)root, row_ptr_, col_idx_, old2new_, keys);
    int rounds = 2;
    while (((int64_t)1 << rounds) < n_ + 1) ++rounds;
    for (int r = 0; r < rounds + 2; ++r) LBFS_LAUNCH(k_val_jump, grid, 256, 0, st, J, n_);
    LBFS_LAUNCH(k_val_status, grid, 256, 0, st, pred, J, n_, (int32_t)root, keys);
    unsigned long long h[5];
    LBFS_CUDA(cudaMemcpyAsync(h, keys, sizeof(h), cudaMemcpyDeviceToHost, st));
    LBFS_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < 5; ++k) {
      const bool pass = h[k] == ~0ull;
      out[k] = pass ? 1 : 0;
      out[5 + k] = pass ? -1 : (k == 2 ? (int64_t)(h[k] & 0xFFFFFFFFull) : (int64_t)h[k]);
    }
  } catch (...) {
    dev_free(J);
    dev_free(keys);
    throw;
  }
  dev_free(J);
  dev_free(keys);
}

}  // namespace lbfs
