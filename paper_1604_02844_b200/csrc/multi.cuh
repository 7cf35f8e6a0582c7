// One process, P GPUs: the partitioned BFS behind lbfs_graph_create(ngpus > 1)
// (multi.cu).
#pragma once

#include <mutex>
#include <vector>

#include "lbfs_internal.cuh"

typedef struct ncclComm* ncclComm_t;

namespace lbfs {

class BfsEngine;

class MultiGraph {
 public:
  // csr: on its own device; partition p goes to devices[p] (nullptr: 0..ngpus-1)
  MultiGraph(const Csr& csr, int ngpus, const int* devices);
  // one partition of a multi-process job (borrowed, not deleted) joined to
  // the other processes' partitions by ncclCommInitRank(id, nparts, rank)
  MultiGraph(BfsEngine* part, const void* nccl_id);
  static void unique_id(void* out128);
  ~MultiGraph();
  MultiGraph(const MultiGraph&) = delete;
  MultiGraph& operator=(const MultiGraph&) = delete;
  // BFS; outputs (original ids) on the first device; d_level may be NULL.
  // gather = false (one local partition only): the owned entries only.
  void run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t, bool gather = true);
  const std::vector<lbfs_layer>& layers() const { return layers_; }
  void last_levels_to_host(int32_t* h_level);
  int64_t n() const { return n_; }
  int64_t nnz() const { return nnz_; }
  int64_t npad() const { return npad_; }
  int ngpus() const { return P_; }
  int local_parts() const { return (int)parts_.size(); }
  int device() const { return dev_.empty() ? 0 : dev_[0]; }
  std::mutex mu;

 private:
  struct Bufs {
    int64_t nwl = 0;
    uint32_t* send = nullptr;   // [P][nwl] marks by owner
    uint32_t* recv = nullptr;   // [P][nwl]
    uint32_t* fsend = nullptr;  // [nwl + 4] owned frontier words + counts
    uint32_t* fgath = nullptr;  // [P][nwl + 4]
    unsigned long long* red = nullptr;
    int32_t* pred = nullptr;    // full-size outputs, combined by all-reduce
    int32_t* level = nullptr;
  };
  void release();
  void alloc_bufs(int p);
  bool own_parts_ = true;
  bool gathered_ = false;  // the last run all-reduced its outputs (b_[0].pred / level hold them)
  int P_ = 0;
  int64_t n_ = 0, nnz_ = 0, npad_ = 0;
  std::vector<int> dev_;
  std::vector<BfsEngine*> parts_;
  std::vector<ncclComm_t> comm_;
  std::vector<cudaStream_t> st_;
  std::vector<cudaEvent_t> ev_;
  std::vector<Bufs> b_;
  std::vector<lbfs_layer> layers_;
};

}  // namespace lbfs
