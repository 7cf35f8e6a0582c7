// Top-down BFS on sm_100a: the hot path of the reference's run_bfs
// (traversal.py:413-422 dispatching to bfs_serial / bfs_parallel_naive /
// _bitmap_bfs, traversal.py:80-389).
//
//   K4 k_init / k_seed    PredecessorArray fill + Bitmap clear + root seed
//                         (traversal.py:42-46, 135-139, 343-347)
//   K1 k_expand_{small,warp,cta}
//                         frontier expansion over CSR, degree-binned
//                         (_frontier_neighbors traversal.py:107-119; the
//                         16-lane Listing-1 gather, traversal.py:297-332)
//   K2 claim()            visited test-and-set: plain L1 load, then 32-bit
//                         atomicOr; the winner writes pred and level
//                         (replaces the unsynchronised OR + restoration of
//                         traversal.py:175-279 and the last-writer pred
//                         scatter of traversal.py:145-147)
//   K3 discover()         next-queue append with warp-aggregated ballot/popc
//                         offsets, binned by degree for the next level
//                         (np.unique merge traversal.py:157-158)
//   K5 BfsEngine::run     level driver (the while loops traversal.py:90,152,366)
//   K6 Counters           per-level LayerStats(input, edges, discovered)
//                         (traversal.py:66-70, 100, 159, 383)
#include <algorithm>
#include <cstring>

#include "bfs_engine.cuh"

namespace lbfs {

constexpr unsigned kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ uint32_t ld_l1(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.ca.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
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

// ---------------------------------------------------------------- K2 claim
// Test-before-atomic: only a vertex whose bit reads clear pays an atomicOr;
// the atomic's previous value decides the unique winner.
__device__ __forceinline__ bool claim(uint32_t* visited, int32_t v) {
  uint32_t* w = visited + (v >> 5);
  const uint32_t bit = 1u << (v & 31);
  if (ld_l1(w) & bit) return false;
  return (atomicOr(w, bit) & bit) == 0;
}

struct Acc {  // per-thread K6 accumulators, reduced once per warp at exit
  unsigned long long disc = 0;
  unsigned long long edges = 0;
};

__device__ __forceinline__ void warp_append(bool take, int32_t val, unsigned long long* tail,
                                            int32_t* q, int lane) {
  const unsigned m = __ballot_sync(kFull, take);
  if (!m) return;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(tail, (unsigned long long)__popc(m));
  base = __shfl_sync(kFull, base, leader);
  if (take) q[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// ---------------------------------------------------------------- K3 discover
// Called by all 32 lanes; `win` lanes own a newly claimed vertex v.
__device__ __forceinline__ void discover(const LevelArgs& a, bool win, int32_t v, int32_t parent,
                                         int lane, Acc& acc) {
  if (!__any_sync(kFull, win)) return;
  int64_t start = 0;
  int32_t deg = 0;
  if (win) {
    start = a.row_ptr[v];
    deg = (int32_t)(a.row_ptr[v + 1] - start);
    a.level[v] = a.next_level;
    a.pred[v] = parent;
    acc.disc += 1;
    acc.edges += (unsigned long long)deg;
  }
  warp_append(win && deg > 0 && deg < kSmallMax, v, &a.next_cnt->bin[kBinSmall], a.next_small, lane);
  warp_append(win && deg >= kSmallMax && deg < kCtaMin, v, &a.next_cnt->bin[kBinWarp], a.next_warp,
              lane);
  const int items = (win && deg >= kCtaMin) ? (deg + kChunk - 1) / kChunk : 0;
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
      a.next_cta[base + off + k] = make_int4(v, k * kChunk, min(kChunk, deg - k * kChunk), 0);
  }
}

__device__ __forceinline__ void flush_acc(const LevelArgs& a, Acc& acc) {
  unsigned long long d = acc.disc, e = acc.edges;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    d += __shfl_xor_sync(kFull, d, o);
    e += __shfl_xor_sync(kFull, e, o);
  }
  if ((threadIdx.x & 31) == 0 && (d | e)) {
    atomicAdd(&a.next_cnt->discovered, d);
    atomicAdd(&a.next_cnt->edges, e);
  }
}

// Warp-cooperative expansion of neighbours [st, en) of parent u: aligned
// 128-bit col_idx loads for the body, scalar peel/remainder (the Listing-1
// peel/body/remainder split, lane.py:100-108). `wid`/`nw` let several warps
// of a CTA share one row.
__device__ __forceinline__ void expand_row(const LevelArgs& a, int32_t u, int64_t st, int64_t en,
                                           int lane, int wid, int nw, Acc& acc) {
  const int64_t al = std::min<int64_t>((st + 3) & ~int64_t(3), en);
  const int64_t bl = std::max<int64_t>(al, en & ~int64_t(3));
  if (wid == 0) {  // peel [st, al) on lanes 0..2, remainder [bl, en) on lanes 8..10
    int64_t j = -1;
    if (lane < 3 && st + lane < al) j = st + lane;
    if (lane >= 8 && lane < 11 && bl + (lane - 8) < en) j = bl + (lane - 8);
    const int32_t v = (j >= 0) ? ld_stream(a.col_idx + j) : 0;
    const bool win = (j >= 0) && claim(a.visited, v);
    discover(a, win, v, u, lane, acc);
  }
  for (int64_t j0 = al + (int64_t)wid * 128; j0 < bl; j0 += (int64_t)nw * 128) {
    const int64_t j = j0 + lane * 4;
    const bool act = j < bl;
    int4 x = make_int4(0, 0, 0, 0);
    if (act) x = ld_stream4(a.col_idx + j);
    bool w0 = false, w1 = false, w2 = false, w3 = false;
    if (act) {
      w0 = claim(a.visited, x.x);
      w1 = claim(a.visited, x.y);
      w2 = claim(a.visited, x.z);
      w3 = claim(a.visited, x.w);
    }
    discover(a, w0, x.x, u, lane, acc);
    discover(a, w1, x.y, u, lane, acc);
    discover(a, w2, x.z, u, lane, acc);
    discover(a, w3, x.w, u, lane, acc);
  }
}

// ---------------------------------------------------------------- K1 bins
// Small bin (deg < 32): a warp takes 32 frontier vertices, scans their
// degrees and walks the concatenated neighbour lists 32 entries at a time,
// so col_idx loads stay dense across vertex boundaries.
__global__ void __launch_bounds__(256) k_expand_small(LevelArgs a, const int32_t* __restrict__ q,
                                                      int64_t nq) {
  __shared__ int32_t s_off[8][32];
  __shared__ int64_t s_start[8][32];
  __shared__ int32_t s_par[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  Acc acc;
  for (int64_t base = gw * 32; base < nq; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t v = -1;
    int64_t st = 0;
    int32_t d = 0;
    if (i < nq) {
      v = q[i];
      st = a.row_ptr[v];
      d = (int32_t)(a.row_ptr[v + 1] - st);
    }
    int incl = d;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    s_off[w][lane] = incl - d;
    s_start[w][lane] = st;
    s_par[w][lane] = v;
    __syncwarp();
    for (int e0 = 0; e0 < total; e0 += 32) {
      const int e = e0 + lane;
      const bool act = e < total;
      int32_t nb = 0, par = 0;
      if (act) {
        int lo = 0;
#pragma unroll
        for (int step = 16; step; step >>= 1)
          if (s_off[w][lo + step] <= e) lo += step;
        nb = ld_stream(a.col_idx + s_start[w][lo] + (e - s_off[w][lo]));
        par = s_par[w][lo];
      }
      const bool win = act && claim(a.visited, nb);
      discover(a, win, nb, par, lane, acc);
    }
    __syncwarp();
  }
  flush_acc(a, acc);
}

// Warp bin (32 <= deg < kCtaMin): one warp per frontier vertex.
__global__ void __launch_bounds__(256) k_expand_warp(LevelArgs a, const int32_t* __restrict__ q,
                                                     int64_t nq) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  Acc acc;
  for (int64_t i = gw; i < nq; i += nwarps) {
    const int32_t u = q[i];
    const int64_t st = a.row_ptr[u], en = a.row_ptr[u + 1];
    expand_row(a, u, st, en, lane, 0, 1, acc);
  }
  flush_acc(a, acc);
}

// CTA bin (deg >= kCtaMin): hubs are split into kChunk-edge items at append
// time; one CTA expands one item with all its warps.
__global__ void __launch_bounds__(256) k_expand_cta(LevelArgs a, const int4* __restrict__ items,
                                                    int64_t nitems) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Acc acc;
  for (int64_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const int4 item = items[it];
    const int64_t st = a.row_ptr[item.x] + item.y;
    expand_row(a, item.x, st, st + item.z, lane, w, nw, acc);
  }
  flush_acc(a, acc);
}

// ---------------------------------------------------------------- K4 init
__global__ void k_init(int32_t* __restrict__ pred, int64_t npad, int32_t* __restrict__ level,
                       int64_t n, uint32_t* __restrict__ visited, int64_t nwords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t; i < npad; i += stride) pred[i] = kSentinel;
  for (int64_t i = t; i < n; i += stride) level[i] = -1;
  for (int64_t i = t; i < nwords; i += stride) visited[i] = 0;
}

__global__ void k_init_vec(int4* __restrict__ pred4, int64_t npad4, int4* __restrict__ level4,
                           int64_t n4, int32_t* __restrict__ level, int64_t n,
                           uint4* __restrict__ visited4, int64_t nwords4, uint32_t* __restrict__ visited,
                           int64_t nwords) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int4 s4 = make_int4(kSentinel, kSentinel, kSentinel, kSentinel);
  const int4 m4 = make_int4(-1, -1, -1, -1);
  for (int64_t i = t; i < npad4; i += stride) pred4[i] = s4;
  for (int64_t i = t; i < n4; i += stride) level4[i] = m4;
  for (int64_t i = 4 * n4 + t; i < n; i += stride) level[i] = -1;
  for (int64_t i = t; i < nwords4; i += stride) visited4[i] = make_uint4(0, 0, 0, 0);
  for (int64_t i = 4 * nwords4 + t; i < nwords; i += stride) visited[i] = 0;
}

__global__ void k_seed(LevelArgs a, int32_t root, Counters* cnt0) {
  const int64_t st = a.row_ptr[root];
  const int32_t deg = (int32_t)(a.row_ptr[root + 1] - st);
  a.visited[root >> 5] |= 1u << (root & 31);
  a.level[root] = 0;
  a.pred[root] = root;
  Counters c{};
  c.discovered = 1;
  c.edges = (unsigned long long)deg;
  if (deg > 0 && deg < kSmallMax) {
    a.next_small[0] = root;
    c.bin[kBinSmall] = 1;
  } else if (deg >= kSmallMax && deg < kCtaMin) {
    a.next_warp[0] = root;
    c.bin[kBinWarp] = 1;
  } else if (deg >= kCtaMin) {
    const int items = (deg + kChunk - 1) / kChunk;
    for (int k = 0; k < items; ++k) a.next_cta[k] = make_int4(root, k * kChunk, min(kChunk, deg - k * kChunk), 0);
    c.bin[kBinCta] = (unsigned long long)items;
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
  row_ptr_ = csr.row_ptr;
  col_idx_ = csr.col_idx;
  owns_csr_ = false;
  LBFS_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  visited_ = dev_alloc<uint32_t>((size_t)nwords_ + 4);
  // Frontier bins, double-buffered. A vertex is discovered once per BFS, so
  // n entries bound the small/warp bins; cta items are bounded by
  // nnz/kChunk + (#vertices with deg >= kCtaMin) <= nnz/kChunk + nnz/kCtaMin.
  cap_small_ = std::max<int64_t>(n_, 1);
  cap_warp_ = std::max<int64_t>(n_, 1);
  cap_cta_ = nnz_ / kChunk + nnz_ / kCtaMin + 2;
  for (int b = 0; b < 2; ++b) {
    q_small_[b] = dev_alloc<int32_t>((size_t)cap_small_);
    q_warp_[b] = dev_alloc<int32_t>((size_t)cap_warp_);
    q_cta_[b] = dev_alloc<int4>((size_t)cap_cta_);
  }
  cnt_ = dev_alloc<Counters>(kCounterRing);
  LBFS_CUDA(cudaMallocHost(&h_cnt_, sizeof(Counters) * kCounterRing));
  for (auto& e : ev_) LBFS_CUDA(cudaEventCreate(&e));
}

BfsEngine::~BfsEngine() {
  cudaStreamSynchronize(stream_);
  dev_free(visited_);
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
  if (owns_csr_) {
    dev_free(row_ptr_);
    dev_free(col_idx_);
  }
  cudaStreamDestroy(stream_);
}

void BfsEngine::adopt_csr() { owns_csr_ = true; }

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
  // K4
  {
    const bool aligned = ((uintptr_t)d_pred % 16 == 0) && ((uintptr_t)d_level % 16 == 0);
    const unsigned grid = clamp_grid((npad_ / 4 + 255) / 256, (int64_t)sm_count_ * 8);
    if (aligned) {
      LBFS_LAUNCH(k_init_vec, grid, 256, 0, st, (int4*)d_pred, npad_ / 4, (int4*)d_level, n_ / 4,
                  d_level, n_, (uint4*)visited_, nwords_ / 4, visited_, nwords_);
    } else {
      LBFS_LAUNCH(k_init, grid, 256, 0, st, d_pred, npad_, d_level, n_, visited_, nwords_);
    }
  }
  LevelArgs a{};
  a.row_ptr = row_ptr_;
  a.col_idx = col_idx_;
  a.visited = visited_;
  a.pred = d_pred;
  a.level = d_level;
  int cur = 0;
  a.next_small = q_small_[cur];
  a.next_warp = q_warp_[cur];
  a.next_cta = q_cta_[cur];
  a.next_cnt = nullptr;
  LBFS_LAUNCH(k_seed, 1, 1, 0, st, a, (int32_t)root, &cnt_[0]);
  LBFS_CUDA(cudaMemcpyAsync(&h_cnt_[0], &cnt_[0], sizeof(Counters), cudaMemcpyDeviceToHost, st));
  LBFS_CUDA(cudaEventRecord(ev_[1], st));
  LBFS_CUDA(cudaStreamSynchronize(st));

  layers_.clear();
  double expand_ms = 0.0;
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
    LBFS_CUDA(cudaEventRecord(ev_[2], st));
    const int64_t ns = (int64_t)c.bin[kBinSmall], nwq = (int64_t)c.bin[kBinWarp],
                  nc = (int64_t)c.bin[kBinCta];
    if (nc > 0)
      LBFS_LAUNCH(k_expand_cta, clamp_grid(nc, (int64_t)sm_count_ * 8), 256, 0, st, a, q_cta_[cur], nc);
    if (nwq > 0)
      LBFS_LAUNCH(k_expand_warp, clamp_grid((nwq + 7) / 8, (int64_t)sm_count_ * 16), 256, 0, st, a,
                  q_warp_[cur], nwq);
    if (ns > 0)
      LBFS_LAUNCH(k_expand_small, clamp_grid((ns + 255) / 256, (int64_t)sm_count_ * 16), 256, 0, st, a,
                  q_small_[cur], ns);
    LBFS_CUDA(cudaEventRecord(ev_[3], st));
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
