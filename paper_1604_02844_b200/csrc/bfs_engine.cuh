// BFS engine: device layout of one graph and the level driver.
#pragma once

#include "lbfs_internal.cuh"

namespace lbfs {

constexpr int32_t kSentinel = LBFS_SENTINEL;  // traversal.py:22
constexpr int kSmallMax = 32;                 // deg < 32: warp-cooperative small bin
constexpr int kCtaMin = 4096;                 // deg >= 4096: CTA bin
constexpr int kChunk = 4096;                  // edges per CTA-bin work item
constexpr int kBinSmall = 0, kBinWarp = 1, kBinCta = 2;
constexpr int kCounterRing = 3;

// Per-level counters (K6). `discovered`/`edges` of level L+1's slot are
// layers[L].discovered and layers[L+1].edges.
struct alignas(64) Counters {
  unsigned long long bin[3];  // next-level bin tails (entries / items)
  unsigned long long discovered;
  unsigned long long edges;   // sum of degree over discovered vertices
  unsigned long long pad[3];
};

struct LevelArgs {
  const int64_t* row_ptr;
  const int32_t* col_idx;
  uint32_t* visited;
  int32_t* pred;
  int32_t* level;
  int32_t next_level;
  Counters* next_cnt;
  int32_t* next_small;
  int32_t* next_warp;
  int4* next_cta;
};

class BfsEngine {
 public:
  explicit BfsEngine(const Csr& csr);  // borrows csr arrays (see adopt_csr)
  ~BfsEngine();
  BfsEngine(const BfsEngine&) = delete;
  BfsEngine& operator=(const BfsEngine&) = delete;

  void adopt_csr();  // take ownership of the borrowed CSR arrays
  void ensure_own_outputs();
  // BFS into device buffers d_pred[pad32(n)], d_level[n]; synchronous.
  void run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t);

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
  int device_ = 0, sm_count_ = 0;
  int64_t n_ = 0, nnz_ = 0, nwords_ = 0, npad_ = 0;
  int64_t* row_ptr_ = nullptr;
  int32_t* col_idx_ = nullptr;
  bool owns_csr_ = false;
  uint32_t* visited_ = nullptr;
  int32_t* q_small_[2] = {nullptr, nullptr};
  int32_t* q_warp_[2] = {nullptr, nullptr};
  int4* q_cta_[2] = {nullptr, nullptr};
  int64_t cap_small_ = 0, cap_warp_ = 0, cap_cta_ = 0;
  Counters* cnt_ = nullptr;
  Counters* h_cnt_ = nullptr;
  int32_t* own_pred_ = nullptr;
  int32_t* own_level_ = nullptr;
  cudaStream_t stream_ = nullptr;
  cudaEvent_t ev_[5] = {};
  std::vector<lbfs_layer> layers_;
};

}  // namespace lbfs

struct lbfs_graph {
  lbfs::BfsEngine* eng = nullptr;
};
