// extern "C" boundary of liblbfs (declared in include/lbfs.h). Every entry
// point converts internal exceptions into LBFS_E* codes plus a thread-local
// message, mirroring the reference's error split: precondition violations
// (assert -> AssertionError in traversal.py:84,133,341 / graph.py:33-37) map to
// LBFS_EINVAL, everything else to a runtime failure.
#include <cstdio>
#include <cstring>

#include "bfs_engine.cuh"

namespace lbfs {

std::atomic<int64_t> g_launches{0};
bool g_sync_each = [] {
  const char* v = getenv("LBFS_SYNC_EACH");
  return v && *v && *v != '0';
}();
bool g_pdl = [] {
  const char* v = getenv("LBFS_NO_PDL");
  return !(v && *v && *v != '0');
}();
void sync_check(cudaStream_t st, const char* kernel, const char* file, int line) {
  const cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    fprintf(stderr, "[lbfs] LBFS_SYNC_EACH: %s failed: %s (%s:%d)\n", kernel, cudaGetErrorString(e), file, line);
    throw_cuda(e, kernel, file, line);
  }
}
static thread_local std::string t_err;

void set_error(const std::string& m) { t_err = m; }

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "%s failed: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
  const int code = (e == cudaErrorMemoryAllocation) ? LBFS_ENOMEM : LBFS_ECUDA;
  throw Failure(code, buf);
}

int current_sm_count() {
  int dev = 0, sms = 0;
  LBFS_CUDA(cudaGetDevice(&dev));
  LBFS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  return sms;
}

template <typename F>
static int guarded(F&& f) {
  try {
    f();
    t_err.clear();
    return LBFS_OK;
  } catch (const Failure& e) {
    t_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    t_err = e.what();
    return LBFS_ECUDA;
  }
}

static void check_ids(int64_t n) {
  if (n < 1) throw_inval("num_vertices must be >= 1");
  if (n > ((int64_t)1 << 31) - 1) throw_inval("num_vertices must fit int32 ids below the sentinel");
}

struct Stream {  // scratch stream for construction calls
  cudaStream_t s = nullptr;
  Stream() { LBFS_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~Stream() { cudaStreamDestroy(s); }
};

}  // namespace lbfs

using namespace lbfs;

extern "C" {

const char* lbfs_last_error(void) { return t_err.c_str(); }

int64_t lbfs_kernel_launch_count(void) { return g_launches.load(); }

int lbfs_host_alloc(int64_t bytes, void** out) {
  return guarded([&] {
    if (!out || bytes < 0) throw_inval("bad arguments");
    void* p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, (size_t)std::max<int64_t>(bytes, 16), cudaHostAllocDefault);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      throw Failure(LBFS_ENOMEM, std::string("cudaHostAlloc failed: ") + cudaGetErrorString(e));
    }
    *out = p;
  });
}

void lbfs_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int lbfs_set_device(int device) {
  return guarded([&] {
    int count = 0;
    LBFS_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw_inval("device out of range");
    LBFS_CUDA(cudaSetDevice(device));
  });
}

int lbfs_device_info_get(int device, lbfs_device_info* out) {
  return guarded([&] {
    if (!out) throw_inval("out is NULL");
    cudaDeviceProp p;
    LBFS_CUDA(cudaGetDeviceProperties(&p, device));
    memset(out, 0, sizeof(*out));
    out->device = device;
    out->sm_count = p.multiProcessorCount;
    out->cc_major = p.major;
    out->cc_minor = p.minor;
    out->l2_bytes = p.l2CacheSize;
    out->hbm_bytes = (int64_t)p.totalGlobalMem;
    out->smem_per_block_optin = (int64_t)p.sharedMemPerBlockOptin;
    strncpy(out->name, p.name, sizeof(out->name) - 1);
  });
}

int lbfs_rmat_edges(int scale, int64_t m, double ab, double a_norm, double c_norm,
                    const uint64_t pcg[4], uint32_t* src_out, uint32_t* dst_out) {
  return guarded([&] {
    if (scale < 1 || scale > 30) throw_inval("scale must be in [1, 30]");
    if (m < 0 || !pcg || (m > 0 && (!src_out || !dst_out))) throw_inval("bad arguments");
    if (m == 0) return;
    Stream s;
    uint32_t* ds = dev_alloc<uint32_t>((size_t)m);
    uint32_t* dd = dev_alloc<uint32_t>((size_t)m);
    try {
      rmat_edges_device(scale, m, ab, a_norm, c_norm, pcg, ds, dd, s.s);
      LBFS_CUDA(cudaMemcpy(src_out, ds, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToHost));
      LBFS_CUDA(cudaMemcpy(dst_out, dd, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToHost));
    } catch (...) {
      dev_free(ds);
      dev_free(dd);
      throw;
    }
    dev_free(ds);
    dev_free(dd);
  });
}

int lbfs_permute_edges(int64_t n, uint64_t seed, uint32_t* src, uint32_t* dst, int64_t m) {
  return guarded([&] {
    check_ids(n);
    if (m < 0 || (m > 0 && (!src || !dst))) throw_inval("bad arguments");
    if (m == 0) return;
    Stream s;
    uint32_t* ds = dev_alloc<uint32_t>((size_t)m);
    uint32_t* dd = dev_alloc<uint32_t>((size_t)m);
    try {
      LBFS_CUDA(cudaMemcpy(ds, src, sizeof(uint32_t) * (size_t)m, cudaMemcpyHostToDevice));
      LBFS_CUDA(cudaMemcpy(dd, dst, sizeof(uint32_t) * (size_t)m, cudaMemcpyHostToDevice));
      permute_edges_device(n, seed, ds, dd, m, s.s);
      LBFS_CUDA(cudaStreamSynchronize(s.s));
      LBFS_CUDA(cudaMemcpy(src, ds, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToHost));
      LBFS_CUDA(cudaMemcpy(dst, dd, sizeof(uint32_t) * (size_t)m, cudaMemcpyDeviceToHost));
    } catch (...) {
      dev_free(ds);
      dev_free(dd);
      throw;
    }
    dev_free(ds);
    dev_free(dd);
  });
}

int lbfs_csr_build(int64_t n, const uint32_t* src, const uint32_t* dst, int64_t m, int symmetrize,
                   int dedup, lbfs_csr** out) {
  return guarded([&] {
    check_ids(n);
    if (!out || m < 0 || (m > 0 && (!src || !dst))) throw_inval("bad arguments");
    Stream s;
    uint32_t* ds = dev_alloc<uint32_t>((size_t)m);
    uint32_t* dd = dev_alloc<uint32_t>((size_t)m);
    auto* h = new lbfs_csr;
    try {
      if (m > 0) {
        LBFS_CUDA(cudaMemcpy(ds, src, sizeof(uint32_t) * (size_t)m, cudaMemcpyHostToDevice));
        LBFS_CUDA(cudaMemcpy(dd, dst, sizeof(uint32_t) * (size_t)m, cudaMemcpyHostToDevice));
      }
      h->c = build_csr_device(n, ds, dd, m, symmetrize != 0, dedup != 0, s.s);
    } catch (...) {
      dev_free(ds);
      dev_free(dd);
      delete h;
      throw;
    }
    dev_free(ds);
    dev_free(dd);
    *out = h;
  });
}

int lbfs_csr_build_rmat(int scale, int edgefactor, double ab, double a_norm, double c_norm,
                        const uint64_t pcg[4], int permute, uint64_t perm_seed, lbfs_csr** out) {
  return guarded([&] {
    if (scale < 1 || scale > 30 || edgefactor < 1 || !pcg || !out) throw_inval("bad arguments");
    const int64_t n = (int64_t)1 << scale;
    const int64_t m = n * edgefactor;
    Stream s;
    uint32_t* ds = dev_alloc<uint32_t>((size_t)m);
    uint32_t* dd = dev_alloc<uint32_t>((size_t)m);
    auto* h = new lbfs_csr;
    try {
      rmat_edges_device(scale, m, ab, a_norm, c_norm, pcg, ds, dd, s.s);
      if (permute) permute_edges_device(n, perm_seed, ds, dd, m, s.s);
      h->c = build_csr_device(n, ds, dd, m, true, true, s.s);
    } catch (...) {
      dev_free(ds);
      dev_free(dd);
      delete h;
      throw;
    }
    dev_free(ds);
    dev_free(dd);
    *out = h;
  });
}

int lbfs_csr_build_lattice(int64_t rows, int64_t cols, int permute, uint64_t perm_seed,
                           lbfs_csr** out) {
  return guarded([&] {
    if (rows < 1 || cols < 1 || !out) throw_inval("bad arguments");
    const int64_t n = rows * cols;
    check_ids(n);
    const int64_t m = rows * (cols - 1) + (rows - 1) * cols;
    Stream s;
    uint32_t* ds = dev_alloc<uint32_t>((size_t)m);
    uint32_t* dd = dev_alloc<uint32_t>((size_t)m);
    auto* h = new lbfs_csr;
    try {
      lattice_edges_device(rows, cols, ds, dd, s.s);
      if (permute) permute_edges_device(n, perm_seed, ds, dd, m, s.s);
      h->c = build_csr_device(n, ds, dd, m, true, true, s.s);
    } catch (...) {
      dev_free(ds);
      dev_free(dd);
      delete h;
      throw;
    }
    dev_free(ds);
    dev_free(dd);
    *out = h;
  });
}

int lbfs_csr_info(const lbfs_csr* csr, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    if (!csr) throw_inval("csr is NULL");
    if (n) *n = csr->c.n;
    if (nnz) *nnz = csr->c.nnz;
  });
}

int lbfs_csr_download(const lbfs_csr* csr, int64_t* row_ptr, int32_t* col_idx) {
  return guarded([&] {
    if (!csr) throw_inval("csr is NULL");
    LBFS_CUDA(cudaSetDevice(csr->c.device));
    if (row_ptr)
      LBFS_CUDA(cudaMemcpy(row_ptr, csr->c.row_ptr, sizeof(int64_t) * (size_t)(csr->c.n + 1),
                           cudaMemcpyDeviceToHost));
    if (col_idx && csr->c.nnz > 0)
      LBFS_CUDA(cudaMemcpy(col_idx, csr->c.col_idx, sizeof(int32_t) * (size_t)csr->c.nnz,
                           cudaMemcpyDeviceToHost));
  });
}

void lbfs_csr_destroy(lbfs_csr* csr) {
  if (!csr) return;
  cudaSetDevice(csr->c.device);
  free_csr(csr->c);
  delete csr;
}

static lbfs_graph* make_graph(const Csr& c, int ngpus, const int* devices, bool partitioned) {
  auto* g = new lbfs_graph;
  try {
    if (partitioned)
      g->multi = new MultiGraph(c, ngpus, devices);
    else
      g->eng = new BfsEngine(c);
  } catch (...) {
    delete g;
    throw;
  }
  return g;
}

int lbfs_graph_create(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz,
                      int ngpus, lbfs_graph** out) {
  return guarded([&] {
    check_ids(n);
    if (!out || !row_ptr || nnz < 0 || (nnz > 0 && !col_idx)) throw_inval("bad arguments");
    if (ngpus < 1) throw_inval("ngpus must be >= 1");
    if (row_ptr[0] != 0 || row_ptr[n] != nnz) throw_inval("row_ptr must start at 0 and end at nnz");
    Csr c;  // temporary upload in original ids; the engine keeps its own layout
    LBFS_CUDA(cudaGetDevice(&c.device));
    c.n = n;
    c.nnz = nnz;
    c.row_ptr = dev_alloc<int64_t>((size_t)n + 1);
    c.col_idx = dev_alloc<int32_t>((size_t)nnz + 4);
    try {
      LBFS_CUDA(cudaMemcpy(c.row_ptr, row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice));
      if (nnz > 0)
        LBFS_CUDA(cudaMemcpy(c.col_idx, col_idx, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice));
      *out = make_graph(c, ngpus, nullptr, ngpus > 1);
    } catch (...) {
      free_csr(c);
      throw;
    }
    free_csr(c);
  });
}

int lbfs_graph_create_from_csr(const lbfs_csr* csr, int ngpus, lbfs_graph** out) {
  return guarded([&] {
    if (!csr || !out) throw_inval("bad arguments");
    if (ngpus < 1) throw_inval("ngpus must be >= 1");
    LBFS_CUDA(cudaSetDevice(csr->c.device));
    *out = make_graph(csr->c, ngpus, nullptr, ngpus > 1);
  });
}

int lbfs_graph_create_partitioned(const lbfs_csr* csr, int ngpus, const int* devices, lbfs_graph** out) {
  return guarded([&] {
    if (!csr || !out) throw_inval("bad arguments");
    LBFS_CUDA(cudaSetDevice(csr->c.device));
    *out = make_graph(csr->c, ngpus, devices, true);
  });
}

void lbfs_graph_destroy(lbfs_graph* g) {
  if (!g) return;
  delete g->multi;  // (borrows g->eng when attached to a partition)
  if (g->eng) {
    cudaSetDevice(g->eng->device());
    delete g->eng;
  }
  delete g;
}

int lbfs_graph_info(const lbfs_graph* g, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    if (n) *n = g->multi ? g->multi->n() : g->eng->n();
    if (nnz) *nnz = g->multi ? g->multi->nnz() : g->eng->nnz();
  });
}

int lbfs_graph_gpus(const lbfs_graph* g, int* ngpus) {
  return guarded([&] {
    if (!g || !ngpus) throw_inval("bad arguments");
    *ngpus = g->multi ? g->multi->ngpus() : 1;
  });
}

static void copy_layers(const std::vector<lbfs_layer>& L, lbfs_layer* out, int64_t cap, int64_t* n_layers) {
  if (n_layers) *n_layers = (int64_t)L.size();
  if (out && cap > 0) {
    const int64_t k = std::min<int64_t>(cap, (int64_t)L.size());
    memcpy(out, L.data(), sizeof(lbfs_layer) * (size_t)k);
  }
}

int lbfs_bfs(lbfs_graph* g, int64_t root, int direction, int32_t* pred_out, int32_t* level_out,
             lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers, lbfs_timing* t_out) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    if (g->multi) {
      MultiGraph& m = *g->multi;
      std::lock_guard<std::mutex> lk(m.mu);
      if (direction != LBFS_DIR_TOP_DOWN) throw_inval("partitioned graphs run top-down");
      LBFS_CUDA(cudaSetDevice(m.device()));
      int32_t* d_pred = dev_alloc<int32_t>((size_t)m.npad());
      lbfs_timing t{};
      try {
        m.run(root, d_pred, nullptr, &t);
        if (pred_out)
          LBFS_CUDA(cudaMemcpy(pred_out, d_pred, sizeof(int32_t) * (size_t)m.npad(), cudaMemcpyDeviceToHost));
        if (level_out) m.last_levels_to_host(level_out);
      } catch (...) {
        dev_free(d_pred);
        throw;
      }
      dev_free(d_pred);
      if (t_out) *t_out = t;
      copy_layers(m.layers(), layers_out, layers_cap, n_layers);
      return;
    }
    BfsEngine& e = *g->eng;
    std::lock_guard<std::mutex> lk(e.mu);
    LBFS_CUDA(cudaSetDevice(e.device()));
    if (root < 0 || root >= e.n()) throw_inval("root out of range");
    e.ensure_own_outputs();
    lbfs_timing t{};
    // the parents are copied while the output pass is still writing later
    // chunks of them (BfsEngine::run_to_host); levels only when asked for
    e.run_to_host(root, direction, pred_out, level_out, &t);
    if (t_out) *t_out = t;
    copy_layers(e.layers(), layers_out, layers_cap, n_layers);
  });
}

int lbfs_bfs_device(lbfs_graph* g, int64_t root, int direction, int32_t* d_pred, int32_t* d_level,
                    lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers,
                    lbfs_timing* t_out) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    if (!d_pred) throw_inval("device pred output must be non-NULL");
    if (g->multi) {
      MultiGraph& m = *g->multi;
      std::lock_guard<std::mutex> lk(m.mu);
      if (direction != LBFS_DIR_TOP_DOWN) throw_inval("partitioned graphs run top-down");
      LBFS_CUDA(cudaSetDevice(m.device()));
      lbfs_timing t{};
      m.run(root, d_pred, d_level, &t);
      if (t_out) *t_out = t;
      copy_layers(m.layers(), layers_out, layers_cap, n_layers);
      return;
    }
    BfsEngine& e = *g->eng;
    std::lock_guard<std::mutex> lk(e.mu);
    LBFS_CUDA(cudaSetDevice(e.device()));
    if (root < 0 || root >= e.n()) throw_inval("root out of range");
    lbfs_timing t{};
    e.run(root, d_pred, d_level, &t, direction);
    if (t_out) *t_out = t;
    copy_layers(e.layers(), layers_out, layers_cap, n_layers);
  });
}

int lbfs_graph_last_layers(lbfs_graph* g, lbfs_layer* out, int64_t cap, int64_t* n_layers) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    if (g->multi) {
      std::lock_guard<std::mutex> lk(g->multi->mu);
      copy_layers(g->multi->layers(), out, cap, n_layers);
      return;
    }
    std::lock_guard<std::mutex> lk(g->eng->mu);
    copy_layers(g->eng->layers(), out, cap, n_layers);
  });
}

int lbfs_graph_last_levels(lbfs_graph* g, int32_t* level_out) {
  return guarded([&] {
    if (!g || !level_out) throw_inval("bad arguments");
    if (g->multi) {
      std::lock_guard<std::mutex> lk(g->multi->mu);
      g->multi->last_levels_to_host(level_out);
      return;
    }
    BfsEngine& e = *g->eng;
    std::lock_guard<std::mutex> lk(e.mu);
    LBFS_CUDA(cudaSetDevice(e.device()));
    e.last_levels_to_host(level_out);
  });
}

/* ---- tree validation on the device ------------------------------------ */

int lbfs_validate_tree_device(lbfs_graph* g, int64_t root, const int32_t* d_pred, int64_t report[10]) {
  return guarded([&] {
    if (!g || !d_pred || !report) throw_inval("bad arguments");
    if (g->multi) throw_inval("validation needs an unpartitioned graph");
    BfsEngine& e = *g->eng;
    std::lock_guard<std::mutex> lk(e.mu);
    LBFS_CUDA(cudaSetDevice(e.device()));
    e.validate_tree(root, d_pred, report);
  });
}

int lbfs_validate_tree(lbfs_graph* g, int64_t root, const int32_t* pred, int64_t report[10]) {
  return guarded([&] {
    if (!g || !pred || !report) throw_inval("bad arguments");
    if (g->multi) throw_inval("validation needs an unpartitioned graph");
    BfsEngine& e = *g->eng;
    std::lock_guard<std::mutex> lk(e.mu);
    LBFS_CUDA(cudaSetDevice(e.device()));
    int32_t* d = dev_alloc<int32_t>((size_t)std::max<int64_t>(e.n(), 1));
    try {
      LBFS_CUDA(cudaMemcpy(d, pred, sizeof(int32_t) * (size_t)e.n(), cudaMemcpyHostToDevice));
      e.validate_tree(root, d, report);
    } catch (...) {
      dev_free(d);
      throw;
    }
    dev_free(d);
  });
}

/* ---- partitioned (multi-GPU) BFS: one partition per process ----------- */

static BfsEngine& part_engine(lbfs_graph* g) {
  if (!g) throw_inval("graph is NULL");
  if (!g->eng) throw_inval("not a single-partition handle (lbfs_part_create)");
  LBFS_CUDA(cudaSetDevice(g->eng->device()));
  return *g->eng;
}

int lbfs_part_create_from_csr(const lbfs_csr* csr, int rank, int nparts, lbfs_graph** out) {
  return guarded([&] {
    if (!csr || !out) throw_inval("bad arguments");
    LBFS_CUDA(cudaSetDevice(csr->c.device));
    auto* g = new lbfs_graph;
    try {
      g->eng = new BfsEngine(csr->c, rank, nparts);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int lbfs_part_create(int64_t n, const int64_t* row_ptr, const int32_t* col_idx, int64_t nnz, int rank,
                     int nparts, lbfs_graph** out) {
  return guarded([&] {
    check_ids(n);
    if (!out || !row_ptr || nnz < 0 || (nnz > 0 && !col_idx)) throw_inval("bad arguments");
    if (row_ptr[0] != 0 || row_ptr[n] != nnz) throw_inval("row_ptr must start at 0 and end at nnz");
    Csr c;
    LBFS_CUDA(cudaGetDevice(&c.device));
    c.n = n;
    c.nnz = nnz;
    c.row_ptr = dev_alloc<int64_t>((size_t)n + 1);
    c.col_idx = dev_alloc<int32_t>((size_t)nnz + 4);
    try {
      LBFS_CUDA(cudaMemcpy(c.row_ptr, row_ptr, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyHostToDevice));
      if (nnz > 0)
        LBFS_CUDA(cudaMemcpy(c.col_idx, col_idx, sizeof(int32_t) * (size_t)nnz, cudaMemcpyHostToDevice));
      auto* g = new lbfs_graph;
      try {
        g->eng = new BfsEngine(c, rank, nparts);
      } catch (...) {
        delete g;
        throw;
      }
      *out = g;
    } catch (...) {
      free_csr(c);
      throw;
    }
    free_csr(c);
  });
}

int lbfs_part_info(const lbfs_graph* g, int* rank, int* nparts, int64_t* nwords, int64_t* n_local,
                   int64_t* nnz_local) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    const BfsEngine& e = *g->eng;
    if (rank) *rank = e.part_rank();
    if (nparts) *nparts = e.nparts();
    if (nwords) *nwords = e.nwords();
    if (n_local) *n_local = e.n_local();
    if (nnz_local) *nnz_local = e.nnz_local();
  });
}

// the caller's stream as given: NULL is the legacy default stream (torch's
// default stream reports cuda_stream == 0), never the library's own stream,
// so the steps stay ordered with the caller's collectives
static cudaStream_t as_stream(lbfs_graph*, void* stream) { return (cudaStream_t)stream; }

int lbfs_part_start(lbfs_graph* g, int64_t root, uint64_t* red, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!red) throw_inval("red is NULL");
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_start(root, as_stream(g, stream), (unsigned long long*)red);
  });
}

int lbfs_part_expand(lbfs_graph* g, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_expand(as_stream(g, stream));
  });
}

int lbfs_part_pack(lbfs_graph* g, uint32_t* send, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!send) throw_inval("send is NULL");
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_pack(send, as_stream(g, stream));
  });
}

int lbfs_part_merge(lbfs_graph* g, const uint32_t* recv, uint32_t* fsend, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!recv || !fsend) throw_inval("NULL buffer");
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_merge(recv, fsend, as_stream(g, stream));
  });
}

int lbfs_part_sync(lbfs_graph* g, const uint32_t* fgath, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!fgath) throw_inval("fgath is NULL");
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_sync(fgath, as_stream(g, stream));
  });
}

int lbfs_part_level_done(lbfs_graph* g, const uint64_t* red_global, lbfs_layer* layer, int* done) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_level_done((const unsigned long long*)red_global, layer, done);
  });
}

int lbfs_part_finish(lbfs_graph* g, int32_t* d_pred, int32_t* d_level, void* stream) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_finish(d_pred, d_level, as_stream(g, stream));
  });
}

int lbfs_nccl_unique_id(uint8_t id[128]) {
  return guarded([&] {
    if (!id) throw_inval("id is NULL");
    MultiGraph::unique_id(id);
  });
}

int lbfs_part_attach_nccl(lbfs_graph* g, const uint8_t id[128], int nranks, int rank) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!id) throw_inval("id is NULL");
    if (g->multi) throw_inval("a communicator is already attached");
    if (nranks != e.nparts() || rank != e.part_rank()) throw_inval("nranks / rank differ from the partition's");
    std::lock_guard<std::mutex> lk(e.mu);
    g->multi = new MultiGraph(&e, id);
  });
}

int lbfs_part_bfs(lbfs_graph* g, int64_t root, int32_t* d_pred, int32_t* d_level, int gather,
                  lbfs_layer* layers_out, int64_t layers_cap, int64_t* n_layers, lbfs_timing* t_out) {
  return guarded([&] {
    if (!g) throw_inval("graph is NULL");
    if (!g->multi || !g->eng) throw_inval("no communicator attached (lbfs_part_attach_nccl)");
    if (!d_pred) throw_inval("device pred output must be non-NULL");
    MultiGraph& m = *g->multi;
    std::lock_guard<std::mutex> lk(m.mu);
    LBFS_CUDA(cudaSetDevice(m.device()));
    lbfs_timing t{};
    m.run(root, d_pred, d_level, &t, gather != 0);
    if (t_out) *t_out = t;
    copy_layers(m.layers(), layers_out, layers_cap, n_layers);
  });
}

int lbfs_part_plan(lbfs_graph* g, int64_t* a2a_words, int64_t* gather_words) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    std::lock_guard<std::mutex> lk(e.mu);
    e.part_plan(a2a_words, gather_words);
  });
}

int lbfs_part_resolve_count(lbfs_graph* g, int64_t* out) {
  return guarded([&] {
    BfsEngine& e = part_engine(g);
    if (!out) throw_inval("out is NULL");
    std::lock_guard<std::mutex> lk(e.mu);
    *out = (int64_t)e.resolve_scanned();
  });
}

}  // extern "C"
