// One process driving P GPUs (lbfs_graph_create(..., ngpus > 1);
// §8e: the 1D partitioned BFS). Partition p lives on device devices[p] as a
// BfsEngine(csr, p, P) (partition.cu: word-cyclic ownership of the
// degree-ordered ids, replicated visited / frontier bitmaps). The library
// owns one NCCL communicator per device (ncclCommInitAll) and drives every
// device from the calling thread: each collective is a ncclGroupStart /
// ncclGroupEnd group with one call per device, so the P ranks of one level
// step enter it together. Per level:
//
//   expand + pack (each device)  -> ncclAlltoAll of the owner slices (marks)
//   merge + compact (each device) -> ncclAllGather of the owned frontier words
//                                   and the local counts
//   sync + done (each device)     -> layer and termination, identical on all
//
// Outputs: every device writes its owned vertices into full-size arrays
// prefilled with SENTINEL / -1; one ncclAllReduce (min for parents, max for
// levels) completes them on every device, and the first device's copy is
// returned. NCCL is loaded at run time (dlopen of libnccl.so.2: the copy torch
// ships, or LBFS_NCCL_LIB), so single-GPU use carries no NCCL dependency.
#include <dlfcn.h>

#include <nccl.h>

#include <chrono>
#include <cstdio>

#include "bfs_engine.cuh"
#include "multi.cuh"

namespace lbfs {

namespace {

struct NcclApi {
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AlltoAll)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string why;
  std::call_once(once, [] {
    const char* env = getenv("LBFS_NCCL_LIB");
    const char* cands[] = {env, "libnccl.so.2",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           "/usr/lib/x86_64-linux-gnu/libnccl.so.2"};
    void* h = nullptr;
    for (const char* c : cands)
      if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) {
      why = "libnccl.so.2 not found (set LBFS_NCCL_LIB)";
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.CommInitAll = reinterpret_cast<decltype(api.CommInitAll)>(sym("ncclCommInitAll"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
    api.AlltoAll = reinterpret_cast<decltype(api.AlltoAll)>(sym("ncclAlltoAll"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
    if (!api.CommInitAll || !api.CommInitRank || !api.GetUniqueId || !api.GroupStart || !api.AllReduce ||
        !api.AllGather || !api.AlltoAll) {
      why = "libnccl.so.2 lacks ncclAlltoAll (needs NCCL >= 2.24)";
      api = NcclApi{};
    }
  });
  if (!api.CommInitAll) throw Failure(LBFS_ENCCL, why);
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw Failure(LBFS_ENCCL, std::string(what) + " failed: " + msg);
  }
}

struct Group {  // ncclGroupStart / ncclGroupEnd around one call per device
  Group() { nccl_check(nccl().GroupStart(), "ncclGroupStart"); }
  ~Group() noexcept(false) { nccl_check(nccl().GroupEnd(), "ncclGroupEnd"); }
};

__global__ void k_copy_words(const uint32_t* __restrict__ a, uint32_t* __restrict__ b, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

}  // namespace

MultiGraph::MultiGraph(const Csr& csr, int ngpus, const int* devices) {
  if (ngpus < 1 || ngpus > 64 || (ngpus & (ngpus - 1)) != 0) throw_inval("ngpus must be a power of two <= 64");
  n_ = csr.n;
  nnz_ = csr.nnz;
  npad_ = pad32(n_);
  P_ = ngpus;
  int count = 0;
  LBFS_CUDA(cudaGetDeviceCount(&count));
  for (int p = 0; p < P_; ++p) {
    const int d = devices ? devices[p] : p;
    if (d < 0 || d >= count) throw_inval("device out of range (" + std::to_string(count) + " visible)");
    dev_.push_back(d);
  }
  const NcclApi& api = nccl();
  comm_.resize(P_);
  nccl_check(api.CommInitAll(comm_.data(), P_, dev_.data()), "ncclCommInitAll");
  parts_.resize(P_, nullptr);
  b_.resize(P_);
  st_.resize(P_, nullptr);
  ev_.resize(2 * P_, nullptr);
  try {
    for (int p = 0; p < P_; ++p) {
      LBFS_CUDA(cudaSetDevice(dev_[p]));
      // the partition is built from a CSR on its own device
      Csr local = csr;
      Csr copy;
      if (dev_[p] != csr.device) {
        copy.device = dev_[p];
        copy.n = csr.n;
        copy.nnz = csr.nnz;
        copy.row_ptr = dev_alloc<int64_t>((size_t)csr.n + 1);
        copy.col_idx = dev_alloc<int32_t>((size_t)csr.nnz + 4);
        LBFS_CUDA(cudaMemcpyPeer(copy.row_ptr, dev_[p], csr.row_ptr, csr.device, sizeof(int64_t) * (size_t)(csr.n + 1)));
        if (csr.nnz)
          LBFS_CUDA(cudaMemcpyPeer(copy.col_idx, dev_[p], csr.col_idx, csr.device, sizeof(int32_t) * (size_t)csr.nnz));
        local = copy;
      }
      try {
        parts_[p] = new BfsEngine(local, p, P_);
      } catch (...) {
        if (copy.row_ptr) free_csr(copy);
        throw;
      }
      if (copy.row_ptr) free_csr(copy);
      alloc_bufs(p);
    }
  } catch (...) {
    release();
    throw;
  }
  LBFS_CUDA(cudaSetDevice(dev_[0]));
}

// (current device = dev_[p])
void MultiGraph::alloc_bufs(int p) {
  const int64_t nwl = parts_[p]->nwords() / P_;
  Bufs& b = b_[p];
  b.nwl = nwl;
  b.send = dev_alloc<uint32_t>((size_t)(P_ * nwl));
  b.recv = dev_alloc<uint32_t>((size_t)(P_ * nwl));
  b.fsend = dev_alloc<uint32_t>((size_t)(nwl + 4));
  b.fgath = dev_alloc<uint32_t>((size_t)(P_ * (nwl + 4)));
  b.red = dev_alloc<unsigned long long>(2);
  b.pred = dev_alloc<int32_t>((size_t)npad_);
  b.level = dev_alloc<int32_t>((size_t)std::max<int64_t>(n_, 1));
  LBFS_CUDA(cudaStreamCreateWithFlags(&st_[p], cudaStreamNonBlocking));
  LBFS_CUDA(cudaEventCreate(&ev_[2 * p]));
  LBFS_CUDA(cudaEventCreate(&ev_[2 * p + 1]));
}

void MultiGraph::unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  memcpy(out128, &id, sizeof(id));
}

MultiGraph::MultiGraph(BfsEngine* part, const void* nccl_id) {
  own_parts_ = false;
  P_ = part->nparts();
  n_ = part->n();
  nnz_ = part->nnz();
  npad_ = pad32(n_);
  dev_.push_back(part->device());
  const NcclApi& api = nccl();
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  comm_.resize(1, nullptr);
  LBFS_CUDA(cudaSetDevice(dev_[0]));
  nccl_check(api.CommInitRank(&comm_[0], P_, id, part->part_rank()), "ncclCommInitRank");
  parts_.push_back(part);
  b_.resize(1);
  st_.resize(1, nullptr);
  ev_.resize(2, nullptr);
  try {
    alloc_bufs(0);
  } catch (...) {
    release();
    throw;
  }
}

void MultiGraph::last_levels_to_host(int32_t* h_level) {
  if (b_.empty() || !gathered_) throw_inval("no gathered BFS has run on this graph");
  LBFS_CUDA(cudaSetDevice(dev_[0]));
  LBFS_CUDA(cudaMemcpyAsync(h_level, b_[0].level, sizeof(int32_t) * (size_t)n_, cudaMemcpyDeviceToHost, st_[0]));
  LBFS_CUDA(cudaStreamSynchronize(st_[0]));
}

void MultiGraph::release() {
  for (int p = 0; p < (int)parts_.size(); ++p) {
    if (p < (int)dev_.size()) cudaSetDevice(dev_[p]);
    if (st_.size() > (size_t)p && st_[p]) cudaStreamSynchronize(st_[p]);
    if (own_parts_) delete parts_[p];
    parts_[p] = nullptr;
    Bufs& b = b_[p];
    dev_free(b.send);
    dev_free(b.recv);
    dev_free(b.fsend);
    dev_free(b.fgath);
    dev_free(b.red);
    dev_free(b.pred);
    dev_free(b.level);
    b = Bufs{};
    if (st_.size() > (size_t)p && st_[p]) cudaStreamDestroy(st_[p]);
    for (int k = 0; k < 2; ++k)
      if (ev_.size() > (size_t)(2 * p + k) && ev_[2 * p + k]) cudaEventDestroy(ev_[2 * p + k]);
  }
  parts_.clear();
  if (nccl().CommDestroy)
    for (auto c : comm_)
      if (c) nccl().CommDestroy(c);
  comm_.clear();
}

MultiGraph::~MultiGraph() { release(); }

void MultiGraph::run(int64_t root, int32_t* d_pred, int32_t* d_level, lbfs_timing* t, bool gather) {
  if (root < 0 || root >= n_) throw_inval("root out of range");
  if (!gather && parts_.size() != 1) throw_inval("gather = 0 needs one partition per process");
  gathered_ = false;
  const int nloc = (int)parts_.size();
  // one rank: every collective is the identity (nothing to send, the gather
  // is this rank's own slice), so none is issued
  const bool solo = P_ == 1;
  const NcclApi& api = nccl();
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t launches0 = g_launches.load();
  auto each = [&](auto&& fn) {
    for (int p = 0; p < nloc; ++p) {
      LBFS_CUDA(cudaSetDevice(dev_[p]));
      fn(p, *parts_[p], b_[p], st_[p]);
    }
  };
  each([&](int p, BfsEngine& e, Bufs& b, cudaStream_t st) {
    LBFS_CUDA(cudaEventRecord(ev_[2 * p], st));
    e.part_start(root, st, b.red);
  });
  if (!solo) {
    Group g;
    each([&](int p, BfsEngine&, Bufs& b, cudaStream_t st) {
      nccl_check(api.AllReduce(b.red, b.red, 2, ncclUint64, ncclSum, comm_[p], st), "ncclAllReduce");
    });
  }
  int done = 0;
  each([&](int, BfsEngine& e, Bufs& b, cudaStream_t) { e.part_level_done(b.red, nullptr, &done); });
  layers_.clear();
  while (!done) {
    // this level's slice sizes (dense bitmaps or sparse id lists; the same
    // on every rank: they follow from the level's global frontier edges)
    int64_t a2a_words = 0, gather_words = 0;
    parts_[0]->part_plan(&a2a_words, &gather_words);
    each([&](int, BfsEngine& e, Bufs& b, cudaStream_t st) {
      e.part_expand(st);
      if (!solo) e.part_pack(b.send, st);
    });
    if (!solo) {
      Group g;
      each([&](int p, BfsEngine&, Bufs& b, cudaStream_t st) {
        nccl_check(api.AlltoAll(b.send, b.recv, (size_t)a2a_words, ncclUint32, comm_[p], st), "ncclAlltoAll");
      });
    }
    each([&](int, BfsEngine& e, Bufs& b, cudaStream_t st) { e.part_merge(b.recv, b.fsend, st); });
    if (!solo) {
      Group g;
      each([&](int p, BfsEngine&, Bufs& b, cudaStream_t st) {
        nccl_check(api.AllGather(b.fsend, b.fgath, (size_t)gather_words, ncclUint32, comm_[p], st), "ncclAllGather");
      });
    }
    each([&](int, BfsEngine& e, Bufs& b, cudaStream_t st) { e.part_sync(solo ? b.fsend : b.fgath, st); });
    lbfs_layer ly{};
    each([&](int p, BfsEngine& e, Bufs&, cudaStream_t) {
      lbfs_layer l{};
      int d = 0;
      e.part_level_done(nullptr, &l, &d);
      if (p == 0) {
        ly = l;
        done = d;
      }
    });
    layers_.push_back(ly);
  }
  if (!gather) {  // this rank's owned entries, straight into the outputs
    each([&](int, BfsEngine& e, Bufs&, cudaStream_t st) { e.part_finish(d_pred, d_level, st); });
  } else {
    // (levels always: lbfs_graph_last_levels reads them later)
    each([&](int, BfsEngine& e, Bufs& b, cudaStream_t st) { e.part_finish(b.pred, b.level, st); });
    if (!solo) {
      Group g;
      each([&](int p, BfsEngine&, Bufs& b, cudaStream_t st) {
        nccl_check(api.AllReduce(b.pred, b.pred, (size_t)npad_, ncclInt32, ncclMin, comm_[p], st), "ncclAllReduce");
        nccl_check(api.AllReduce(b.level, b.level, (size_t)n_, ncclInt32, ncclMax, comm_[p], st), "ncclAllReduce");
      });
    }
  }
  gathered_ = gather;
  each([&](int p, BfsEngine&, Bufs& b, cudaStream_t st) {
    if (p == 0 && gather) {
      LBFS_CUDA(cudaMemcpyAsync(d_pred, b.pred, sizeof(int32_t) * (size_t)npad_, cudaMemcpyDeviceToDevice, st));
      if (d_level)
        LBFS_CUDA(cudaMemcpyAsync(d_level, b.level, sizeof(int32_t) * (size_t)n_, cudaMemcpyDeviceToDevice, st));
    }
    LBFS_CUDA(cudaEventRecord(ev_[2 * p + 1], st));
  });
  float ms_max = 0.f;
  each([&](int p, BfsEngine&, Bufs&, cudaStream_t) {
    LBFS_CUDA(cudaEventSynchronize(ev_[2 * p + 1]));
    float ms = 0.f;
    LBFS_CUDA(cudaEventElapsedTime(&ms, ev_[2 * p], ev_[2 * p + 1]));
    ms_max = std::max(ms_max, ms);
  });
  LBFS_CUDA(cudaSetDevice(dev_[0]));
  if (t) {
    *t = lbfs_timing{};
    t->bfs_ms = ms_max;  // per device CUDA-event time, max over devices
    t->levels = (int64_t)layers_.size();
    t->kernel_launches = g_launches.load() - launches0;
    for (auto& l : layers_) {
      t->edges += l.edges;
      t->reached += l.input;
    }
    t->d2h_ms = 0.0;
    (void)t0;
  }
}

}  // namespace lbfs
