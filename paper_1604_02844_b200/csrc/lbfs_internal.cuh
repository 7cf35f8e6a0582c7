// Internal declarations shared by the CUDA translation units of liblbfs.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "lbfs.h"

namespace lbfs {

// Internal failures are C++ exceptions carrying an LBFS_E* code; every
// extern "C" entry point catches them and returns the code.
struct Failure : std::runtime_error {
  int code;
  Failure(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);
[[noreturn]] inline void throw_inval(const std::string& m) { throw Failure(LBFS_EINVAL, m); }

#define LBFS_CUDA(call)                                                    \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) ::lbfs::throw_cuda(e_, #call, __FILE__, __LINE__); \
  } while (0)

// Counted launch: every kernel the library issues goes through this macro
// so bench.py can report gpu_launches.
extern std::atomic<int64_t> g_launches;
extern bool g_sync_each;  // LBFS_SYNC_EACH=1 (debug): synchronise after every launch, name the failing kernel
void sync_check(cudaStream_t st, const char* kernel, const char* file, int line);
#define LBFS_LAUNCH(kernel, grid, block, smem, stream, ...)               \
  do {                                                                     \
    kernel<<<(grid), (block), (smem), (stream)>>>(__VA_ARGS__);            \
    ::lbfs::g_launches.fetch_add(1, std::memory_order_relaxed);            \
    LBFS_CUDA(cudaGetLastError());                                         \
    if (::lbfs::g_sync_each) ::lbfs::sync_check((stream), #kernel, __FILE__, __LINE__); \
  } while (0)

// Programmatic dependent launch: the kernel may start (its CTAs take the SMs the
// previous kernel of the stream frees, and run their prologue) before that
// kernel has completed; it calls griddep_wait() before touching anything the
// previous kernel wrote. Only for a kernel that directly follows another
// kernel on the stream (LBFS_NO_PDL=1: plain launches).
extern bool g_pdl;
#define LBFS_LAUNCH_PDL(KERNEL, GRID, BLOCK, SMEM, STREAM, ...)                          \
  do {                                                                                  \
    if (::lbfs::g_pdl) {                                                                \
      cudaLaunchConfig_t cfg_{};                                                        \
      cfg_.gridDim = dim3(GRID);                                                        \
      cfg_.blockDim = dim3(BLOCK);                                                      \
      cfg_.dynamicSmemBytes = (size_t)(SMEM);                                           \
      cfg_.stream = (STREAM);                                                           \
      cudaLaunchAttribute at_[1];                                                       \
      at_[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;                   \
      at_[0].val.programmaticStreamSerializationAllowed = 1;                            \
      cfg_.attrs = at_;                                                                 \
      cfg_.numAttrs = 1;                                                                \
      LBFS_CUDA(cudaLaunchKernelEx(&cfg_, KERNEL, __VA_ARGS__));                        \
      ::lbfs::g_launches.fetch_add(1, std::memory_order_relaxed);                       \
      if (::lbfs::g_sync_each) ::lbfs::sync_check((STREAM), #KERNEL, __FILE__, __LINE__); \
    } else {                                                                            \
      LBFS_LAUNCH(KERNEL, GRID, BLOCK, SMEM, STREAM, __VA_ARGS__);                      \
    }                                                                                   \
  } while (0)

void set_error(const std::string& m);

template <typename T>
T* dev_alloc(size_t count) {
  if (count == 0) count = 1;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, count * sizeof(T));
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    throw Failure(LBFS_ENOMEM, std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) +
                                   " bytes) failed: " + cudaGetErrorString(e));
  }
  return static_cast<T*>(p);
}

inline void dev_free(void* p) {
  if (p) cudaFree(p);
}

inline int64_t pad32(int64_t n) { return (n + 31) / 32 * 32; }

int current_sm_count();

// ---------------------------------------------------------------- construct
struct PcgJump {  // affine map s -> mult*s + plus (mod 2^128), as lo/hi words
  uint64_t mult_lo, mult_hi, plus_lo, plus_hi;
};

// Device CSR in original vertex ids (the reference CsrGraph contents).
struct Csr {
  int device = 0;
  int64_t n = 0, nnz = 0;
  int64_t* row_ptr = nullptr;  // [n+1]
  int32_t* col_idx = nullptr;  // [nnz], 256-B aligned base
};

void rmat_edges_device(int scale, int64_t m, double ab, double a_norm, double c_norm,
                       const uint64_t pcg[4], uint32_t* d_src, uint32_t* d_dst, cudaStream_t st);
void permute_edges_device(int64_t n, uint64_t seed, uint32_t* d_src, uint32_t* d_dst, int64_t m,
                          cudaStream_t st);
void lattice_edges_device(int64_t rows, int64_t cols, uint32_t* d_src, uint32_t* d_dst,
                          cudaStream_t st);
// Consumes (frees) nothing; d_src/d_dst stay owned by the caller.
Csr build_csr_device(int64_t n, const uint32_t* d_src, const uint32_t* d_dst, int64_t m,
                     bool symmetrize, bool dedup, cudaStream_t st);
void free_csr(Csr& c);

}  // namespace lbfs

struct lbfs_csr {
  lbfs::Csr c;
};
