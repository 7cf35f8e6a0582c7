// Traversal layout of a graph (built once, not timed — the analogue of the
// reference's 64-byte-aligned CsrGraph arrays, graph.py:88-93).
//
// Vertices are relabelled by descending degree (ties by original id), rows
// are gathered in that order with neighbours mapped to internal ids and
// sorted ascending. Bins become id ranges [0,t_cta) / [t_cta,t_warp) /
// [t_warp,t_nz), and the visited words of high-degree vertices, which
// receive most probes, form a small bitmap prefix.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "bfs_engine.cuh"

namespace lbfs {

__global__ void k_degree_keys(const int64_t* __restrict__ rp, int64_t n, uint32_t* __restrict__ key,
                              int32_t* __restrict__ ids) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = rp[v + 1] - rp[v];
    key[v] = 0x7FFFFFFFu - (uint32_t)d;  // ascending key == descending degree
    ids[v] = (int32_t)v;
  }
}

__global__ void k_invert(const int32_t* __restrict__ new2old, int64_t n, int32_t* __restrict__ old2new,
                         const uint32_t* __restrict__ key, int64_t* __restrict__ deg64) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    old2new[new2old[i]] = (int32_t)i;
    deg64[i] = (int64_t)(0x7FFFFFFFu - key[i]);
  }
}

// thresholds over the descending degree sequence: t[k] = #vertices with
// deg >= k for k in [1, kSmallMax + 1], t[0] = #vertices with deg >= kCtaMin
constexpr int kNumThresh = kSmallMax + 2;
__global__ void k_thresholds(const int64_t* __restrict__ deg, int64_t n, int32_t* __restrict__ t) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int k = 0; k < kNumThresh; ++k) {
      const int64_t X = (k == 0) ? kCtaMin : k;
      const bool here = deg[i] >= X;
      const bool next = (i + 1 < n) && deg[i + 1] >= X;
      if (here && !next) t[k] = (int32_t)(i + 1);
    }
  }
}

// Partitioned layout (nparts > 1): rank g owns the internal ids of bitmap
// words w with w % nparts == g; its local row l is internal id
// ((l/32)*nparts + g)*32 + l%32. Local degrees / original ids of the owned
// rows (rows past n are empty padding).
__global__ void k_local_rows(const int64_t* __restrict__ deg64, const int32_t* __restrict__ new2old, int64_t n,
                             int64_t n_loc, int part_log, int rank, int64_t* __restrict__ deg_loc,
                             int32_t* __restrict__ new2old_loc) {
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n_loc;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = ((((l >> 5) << part_log) | rank) << 5) | (l & 31);
    deg_loc[l] = v < n ? deg64[v] : 0;
    new2old_loc[l] = v < n ? new2old[v] : 0;
  }
}

// warp per internal row: gather the original row, map neighbours to internal ids
__global__ void k_gather_rows(const int64_t* __restrict__ old_rp, const int32_t* __restrict__ old_ci,
                              const int64_t* __restrict__ new_rp, const int32_t* __restrict__ new2old,
                              const int32_t* __restrict__ old2new, int64_t n, int32_t* __restrict__ new_ci) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t o = new2old[r];
    const int64_t src = old_rp[o], len = old_rp[o + 1] - src, dst = new_rp[r];
    for (int64_t k = lane; k < len; k += 32) new_ci[dst + k] = old2new[old_ci[src + k]];
  }
}

struct SubBase {
  int64_t base;
  __host__ __device__ int operator()(int64_t x) const { return (int)(x - base); }
};

static unsigned grid_of(int64_t work, int threads = 256) {
  const int64_t cap = (int64_t)current_sm_count() * 32;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + threads - 1) / threads, cap));
}

__global__ void k_first_nbr(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t n,
                            int32_t* __restrict__ out) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = rp[v] < rp[v + 1] ? ci[rp[v]] : 0;
}

void BfsEngine::build_layout(const Csr& csr) {
  cudaStream_t st = stream_;
  const int64_t n = csr.n;
  const int64_t nl = n_loc_;  // rows of this rank (== n unpartitioned)
  // 1. degree-descending order
  uint32_t* key = dev_alloc<uint32_t>((size_t)n);
  uint32_t* key_s = dev_alloc<uint32_t>((size_t)n);
  int32_t* ids = dev_alloc<int32_t>((size_t)n);
  new2old_ = dev_alloc<int32_t>((size_t)n);
  old2new_ = dev_alloc<int32_t>((size_t)pad32(n) + 4);  // padded: k_finalize reads whole int4 of it
  LBFS_LAUNCH(k_degree_keys, grid_of(n), 256, 0, st, csr.row_ptr, n, key, ids);
  size_t tmp_bytes = 0;
  LBFS_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key_s, ids, new2old_, n, 0, 32, st));
  void* tmp = dev_alloc<uint8_t>(tmp_bytes);
  LBFS_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key_s, ids, new2old_, n, 0, 32, st));
  LBFS_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp);
  dev_free(key);
  dev_free(ids);
  // 2. inverse map, internal degrees, row_ptr
  int64_t* deg64 = dev_alloc<int64_t>((size_t)n + 1);
  LBFS_LAUNCH(k_invert, grid_of(n), 256, 0, st, new2old_, n, old2new_, key_s, deg64);
  LBFS_CUDA(cudaMemsetAsync(deg64 + n, 0, sizeof(int64_t), st));
  dev_free(key_s);
  // 2b. the rows this rank owns (all rows when unpartitioned)
  int64_t* deg_loc = deg64;
  if (nparts_ > 1) {
    deg_loc = dev_alloc<int64_t>((size_t)nl + 1);
    new2old_loc_ = dev_alloc<int32_t>((size_t)nl);
    LBFS_LAUNCH(k_local_rows, grid_of(nl), 256, 0, st, deg64, new2old_, n, nl, part_log_, part_rank_, deg_loc,
                new2old_loc_);
    LBFS_CUDA(cudaMemsetAsync(deg_loc + nl, 0, sizeof(int64_t), st));
  } else {
    new2old_loc_ = new2old_;
  }
  int32_t* d_t3 = dev_alloc<int32_t>(kNumThresh);
  LBFS_CUDA(cudaMemsetAsync(d_t3, 0, kNumThresh * sizeof(int32_t), st));
  LBFS_LAUNCH(k_thresholds, grid_of(nl), 256, 0, st, deg_loc, nl, d_t3);
  int32_t h_t[kNumThresh];
  LBFS_CUDA(cudaMemcpyAsync(h_t, d_t3, sizeof(h_t), cudaMemcpyDeviceToHost, st));
  row_ptr_ = dev_alloc<int64_t>((size_t)nl + 1);
  tmp_bytes = 0;
  LBFS_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, deg_loc, row_ptr_, nl + 1, st));
  tmp = dev_alloc<uint8_t>(tmp_bytes);
  LBFS_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, deg_loc, row_ptr_, nl + 1, st));
  LBFS_CUDA(cudaStreamSynchronize(st));
  dev_free(tmp);
  if (deg_loc != deg64) dev_free(deg_loc);
  dev_free(deg64);
  dev_free(d_t3);
  t_cta_ = h_t[0];
  t_warp_ = std::max(h_t[kSmallMax], t_cta_);
  t_nz_ = std::max(h_t[1], t_warp_);
  std::vector<int64_t> h_rp((size_t)nl + 1);
  LBFS_CUDA(cudaMemcpyAsync(h_rp.data(), row_ptr_, sizeof(int64_t) * (size_t)(nl + 1), cudaMemcpyDeviceToHost, st));
  LBFS_CUDA(cudaStreamSynchronize(st));
  nnz_loc_ = h_rp[(size_t)nl];
  // 3. gather + map rows (16-byte aligned base, padded for int4 over-reads)
  col_idx_ = dev_alloc<int32_t>((size_t)nnz_loc_ + 8);
  int32_t* unsorted = dev_alloc<int32_t>((size_t)nnz_loc_ + 8);
  LBFS_LAUNCH(k_gather_rows, grid_of(nl * 32), 256, 0, st, csr.row_ptr, csr.col_idx, row_ptr_, new2old_loc_,
              old2new_, nl, unsorted);
  // 4. sort every row ascending; CUB's segmented sort takes int sizes, so go
  //    in row ranges of < 2^30 entries
  const int64_t kMaxItems = (int64_t)1 << 30;
  int64_t r0 = 0;
  while (r0 < nl) {
    int64_t r1 = r0 + 1;
    // extend the range while it stays below kMaxItems entries (binary search)
    int64_t lo = r0 + 1, hi = nl;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) / 2;
      if (h_rp[mid] - h_rp[r0] <= kMaxItems) lo = mid; else hi = mid - 1;
    }
    r1 = std::max(lo, r0 + 1);
    const int64_t base = h_rp[r0];
    const int items = (int)(h_rp[r1] - base);
    if (items > 0) {
      cub::TransformInputIterator<int, SubBase, const int64_t*> beg(row_ptr_ + r0, SubBase{base});
      cub::TransformInputIterator<int, SubBase, const int64_t*> end(row_ptr_ + r0 + 1, SubBase{base});
      tmp_bytes = 0;
      LBFS_CUDA(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp_bytes, unsorted + base, col_idx_ + base,
                                                   items, (int)(r1 - r0), beg, end, st));
      tmp = dev_alloc<uint8_t>(tmp_bytes);
      LBFS_CUDA(cub::DeviceSegmentedSort::SortKeys(tmp, tmp_bytes, unsorted + base, col_idx_ + base, items,
                                                   (int)(r1 - r0), beg, end, st));
      LBFS_CUDA(cudaStreamSynchronize(st));
      dev_free(tmp);
    }
    r0 = r1;
  }
  dev_free(unsorted);
  // 5. degree classes of the small region (deg in [1, kSmallMax))
  ClassTable ct{};
  for (int d = 1; d <= kSmallMax + 1; ++d) ct.T[d] = h_t[d];
  ct.T[0] = (int32_t)nl;
  for (int d = 1; d <= kSmallMax; ++d) ct.base[d] = h_rp[(size_t)(d <= kSmallMax ? h_t[std::min(d + 1, kSmallMax + 1)] : 0)];
  classes_ = dev_alloc<ClassTable>(1);
  LBFS_CUDA(cudaMemcpyAsync(classes_, &ct, sizeof(ct), cudaMemcpyHostToDevice, st));
  // 6. dense tasks over the small region: kDenseTask-element ranges inside a class
  std::vector<DenseTask> tasks;
  for (int d = kSmallMax - 1; d >= 1; --d) {
    const int64_t lo = ct.T[d + 1], hi = ct.T[d];
    if (hi <= lo) continue;
    const int64_t e0 = ct.base[d], e1 = ct.base[d] + (hi - lo) * d;
    for (int64_t p = e0; p < e1; p += kDenseTask)
      tasks.push_back(DenseTask{p, (int32_t)std::min<int64_t>(kDenseTask, e1 - p), d});
  }
  n_dense_tasks_ = (int64_t)tasks.size();
  dense_tasks_ = dev_alloc<DenseTask>(std::max<size_t>(tasks.size(), 1));
  if (!tasks.empty())
    LBFS_CUDA(cudaMemcpyAsync(dense_tasks_, tasks.data(), sizeof(DenseTask) * tasks.size(), cudaMemcpyHostToDevice, st));
  // 7. heavy levels: first neighbour of each row (the parent candidate of a
  // vertex found by a blind OR) and the side entries of the big-row windows
  if (nparts_ == 1) {
    first_nbr_ = dev_alloc<int32_t>((size_t)std::max<int64_t>(nl, 1));
    LBFS_LAUNCH(k_first_nbr, clamp_grid((nl + 255) / 256, 148 * 16), 256, 0, st, row_ptr_, col_idx_, nl, first_nbr_);
  }
  // 7. heavy-level sweep: side entries of the big-row region's windows
  e_big_ = h_rp[(size_t)t_warp_];
  e_nz_ = h_rp[(size_t)t_nz_];
  n_win_all_ = (e_nz_ + kSweepWindow - 1) / kSweepWindow;
  w_small0_ = e_big_ / kSweepWindow;
  if (n_win_all_ > w_small0_) {
    const int64_t nsw = n_win_all_ - w_small0_;
    svmask_ = dev_alloc<uint4>((size_t)nsw);
    sdesc_ = dev_alloc<uint2>((size_t)nsw);
  }
  n_side_win_ = t_warp_ > 0 ? (e_big_ + kSweepWindow - 1) / kSweepWindow : 0;
  if (n_side_win_ > 0) {
    side_ = dev_alloc<uint2>((size_t)n_side_win_);
    LBFS_LAUNCH(k_side_table, clamp_grid((n_side_win_ + 255) / 256, 148 * 16), 256, 0, st, row_ptr_, t_warp_,
                n_side_win_, side_);
  }
  if (sdesc_)
    LBFS_LAUNCH(k_small_desc, clamp_grid((n_win_all_ - w_small0_ + 255) / 256, 148 * 16), 256, 0, st, classes_, e_big_,
                e_nz_, w_small0_, n_win_all_ - w_small0_, sdesc_);
  LBFS_CUDA(cudaStreamSynchronize(st));
}

}  // namespace lbfs
