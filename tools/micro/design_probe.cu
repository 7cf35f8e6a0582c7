// Microbenchmarks (dev) behind the round-2 level-driver design:
//   1. CUDA graph conditional WHILE loop: per-iteration cost of an empty body,
//      of a body with one IF node, and of a body launching a persistent kernel
//   2. thread-block cluster barrier latency (cluster 8 and 16 CTAs x 1024 thr)
//   3. dependent-chain latency: DSMEM atom.or to a peer CTA vs global atom.or (L2)
//   4. grid barrier over 148 CTAs (one global arrival counter) for comparison
//   5. random ld.global.cg throughput over a 2 MiB bitmap (vs red.or, scatter_ops.cu)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      printf("%s failed: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__);               \
      return 1;                                                                                \
    }                                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// ---------------------------------------------------------------- 1. graphs
__global__ void k_dec(int* ctr, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0) {
    int c = --(*ctr);
    cudaGraphSetConditional(h, c > 0 ? 1u : 0u);
  }
}
__global__ void k_set_if(int* ctr, cudaGraphConditionalHandle hif) {
  if (threadIdx.x == 0) cudaGraphSetConditional(hif, (*ctr & 1) ? 1u : 0u);
}
__global__ void __launch_bounds__(1024, 1) k_persist(int* sink) {
  extern __shared__ uint32_t s[];
  if (threadIdx.x == 0) s[0] = blockIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && s[0] == 0xFFFFFFFF) *sink = 1;
}
__global__ void k_init_ctr(int* ctr, int v) { *ctr = v; }

static int graph_probe() {
  int* ctr;
  int* sink;
  CK(cudaMalloc(&ctr, 4));
  CK(cudaMalloc(&sink, 4));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  CK(cudaFuncSetAttribute(k_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  for (int variant = 0; variant < 4; ++variant) {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw;
    CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = hw;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wn;
    CK(cudaGraphAddNode(&wn, g, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];
    cudaGraphNode_t prev = nullptr;
    auto add_kernel = [&](cudaGraph_t gr, void* fn, dim3 grid, dim3 block, int smem, void** args,
                          cudaGraphNode_t* dep) -> cudaGraphNode_t {
      cudaKernelNodeParams kp = {};
      kp.func = fn;
      kp.gridDim = grid;
      kp.blockDim = block;
      kp.sharedMemBytes = smem;
      kp.kernelParams = args;
      cudaGraphNode_t n;
      if (cudaGraphAddKernelNode(&n, gr, dep, dep ? 1 : 0, &kp) != cudaSuccess) printf("add kernel failed\n");
      return n;
    };
    void* a_dec[] = {&ctr, &hw};
    if (variant >= 1) {  // persistent kernel in the body (variant 1: direct; 2: inside IF; 3: IF skipped half)
      if (variant == 1) {
        void* a_p[] = {&sink};
        prev = add_kernel(body, (void*)k_persist, dim3(148), dim3(1024), 200 * 1024, a_p, nullptr);
      } else {
        cudaGraphConditionalHandle hif;
        CK(cudaGraphConditionalHandleCreate(&hif, body, 0, cudaGraphCondAssignDefault));
        void* a_s[] = {&ctr, &hif};
        cudaGraphNode_t sn = add_kernel(body, (void*)k_set_if, dim3(1), dim3(32), 0, a_s, nullptr);
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = hif;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t in;
        CK(cudaGraphAddNode(&in, body, &sn, 1, &ip));
        void* a_p[] = {&sink};
        if (variant == 2) add_kernel(ip.conditional.phGraph_out[0], (void*)k_persist, dim3(148), dim3(1024), 200 * 1024, a_p, nullptr);
        else add_kernel(ip.conditional.phGraph_out[0], (void*)k_persist, dim3(1), dim3(32), 16, a_p, nullptr);
        prev = in;
      }
    }
    add_kernel(body, (void*)k_dec, dim3(1), dim3(32), 0, a_dec, prev ? &prev : nullptr);
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    const int iters = 1000;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 3; ++rep) {
      k_init_ctr<<<1, 1, 0, st>>>(ctr, iters);
      CK(cudaEventRecord(a, st));
      CK(cudaGraphLaunch(ex, st));
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const char* names[] = {"WHILE{dec}", "WHILE{persist148x1024,dec}", "WHILE{setif,IF{persist148},dec}",
                           "WHILE{setif,IF{tiny},dec}"};
    printf("graph %-36s %.2f us/iter\n", names[variant], ms * 1e3 / iters);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
  }
  // plain stream launches for comparison
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaEventRecord(a, st));
      for (int i = 0; i < 1000; ++i) k_persist<<<148, 1024, 200 * 1024, st>>>(sink);
      CK(cudaEventRecord(b, st));
      CK(cudaEventSynchronize(b));
    }
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("stream back-to-back persist148x1024      %.2f us/launch\n", ms);
  }
  return 0;
}

// ---------------------------------------------------------------- 2/3. clusters
__device__ __forceinline__ void cluster_bar() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__global__ void __launch_bounds__(1024, 1) k_cluster_bar(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cluster_bar();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[blockIdx.x / cl.num_blocks()] = t1 - t0;
}
__global__ void __launch_bounds__(1024, 1) k_dsmem_lat(int iters, unsigned long long* out, uint32_t* gbuf) {
  extern __shared__ uint32_t s[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = 0;
  cl.sync();
  if (cl.block_rank() == 0 && threadIdx.x == 0) {
    uint32_t base = (uint32_t)__cvta_generic_to_shared(s), rb;
    const uint32_t peer = cl.num_blocks() - 1;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(base), "r"(peer));
    uint32_t v = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t old;
      asm volatile("atom.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(rb + ((v & 255) << 2)), "r"(1u) : "memory");
      v += old + 1;
    }
    unsigned long long t1 = clock64();
    uint32_t gv = 0;
    for (int i = 0; i < iters; ++i) {
      uint32_t old = atomicOr(gbuf + ((gv * 97) & 65535), 1u);
      gv += old + 1;
    }
    unsigned long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
      uint32_t old = __ldcg(gbuf + ((gv * 97) & 65535));
      gv += old + 1;
    }
    unsigned long long t3 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t1;
    out[2] = t3 - t2;
    out[3] = v + gv;
  }
  cl.sync();
}

static int cluster_probe() {
  unsigned long long* out;
  uint32_t* gbuf;
  CK(cudaMalloc(&out, 4096));
  CK(cudaMalloc(&gbuf, 1 << 20));
  CK(cudaMemset(gbuf, 0, 1 << 20));
  CK(cudaFuncSetAttribute(k_cluster_bar, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dsmem_lat, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(k_dsmem_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  for (int cs : {2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void*)k_cluster_bar, &cfg);
    const int iters = 10000;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster_bar, iters, out);
    CK(cudaDeviceSynchronize());
    if (e != cudaSuccess) {
      printf("cluster %d: launch failed %s\n", cs, cudaGetErrorString(e));
      continue;
    }
    unsigned long long cyc;
    CK(cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost));
    printf("cluster %2d x1024: barrier %.0f cycles (%.3f us @1.965GHz); max active clusters %d\n", cs,
           (double)cyc / iters, (double)cyc / iters / 1965.0, ncl);
    cfg.dynamicSmemBytes = 64 * 1024;
    e = cudaLaunchKernelEx(&cfg, k_dsmem_lat, 1000, out, gbuf);
    CK(cudaDeviceSynchronize());
    unsigned long long r[4];
    CK(cudaMemcpy(r, out, 32, cudaMemcpyDeviceToHost));
    printf("   dependent atom latency: dsmem %.0f cyc, global atomicOr %.0f cyc, ld.cg %.0f cyc\n", r[0] / 1000.0,
           r[1] / 1000.0, r[2] / 1000.0);
  }
  return 0;
}

// ---------------------------------------------------------------- 4. grid barrier
__global__ void k_grid_bar(unsigned* count, unsigned* gen, int iters, unsigned long long* out) {
  unsigned g = 0;
  if (threadIdx.x == 0) g = *(volatile unsigned*)gen;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned r;
      asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(r) : "l"(count) : "memory");
      if (r == gridDim.x - 1) {
        *(volatile unsigned*)count = 0;
        asm volatile("red.add.release.gpu.global.u32 [%0], 1;" ::"l"(gen) : "memory");
      } else {
        unsigned v;
        do {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(gen) : "memory");
        } while (v == g);
      }
      ++g;
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

// ---------------------------------------------------------------- 5. random loads
constexpr int K = 256;
__global__ void __launch_bounds__(1024) k_rand_ld(const uint32_t* bm, uint32_t mask_words, uint32_t seed, uint32_t* out) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x, acc = 0;
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    uint32_t v = hsh(t * K + k + seed);
    acc ^= __ldcg(bm + ((v >> 5) & mask_words));
  }
  if (acc == 0x12345678) out[0] = acc;
}
__global__ void __launch_bounds__(1024) k_rand_red(uint32_t* bm, uint32_t mask_words, uint32_t seed) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    uint32_t v = hsh(t * K + k + seed);
    asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(bm + ((v >> 5) & mask_words)), "r"(1u << (v & 31)) : "memory");
  }
}
__global__ void __launch_bounds__(1024) k_rand_red_shared(uint32_t* out, uint32_t seed, int words) {
  extern __shared__ uint32_t s[];
  for (int i = threadIdx.x; i < words; i += blockDim.x) s[i] = 0;
  __syncthreads();
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(s);
#pragma unroll 8
  for (int k = 0; k < K; ++k) {
    uint32_t v = hsh(t * K + k + seed);
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(base + ((v >> 5) % words) * 4), "r"(1u << (v & 31)) : "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[seed % words];
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("%s, %d SMs, L2 %d MB\n", p.name, p.multiProcessorCount, p.l2CacheSize >> 20);
  if (graph_probe()) return 1;
  if (cluster_probe()) return 1;
  unsigned* bar;
  unsigned long long* out;
  uint32_t *bm, *o2;
  CK(cudaMalloc(&bar, 64));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&bm, 2 << 20));
  CK(cudaMalloc(&o2, 4096));
  CK(cudaMemset(bar, 0, 64));
  CK(cudaMemset(bm, 0, 2 << 20));
  for (int grid : {16, 32, 148}) {
    k_grid_bar<<<grid, 512>>>(bar, bar + 8, 10000, out);
    CK(cudaDeviceSynchronize());
    unsigned long long cyc;
    CK(cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost));
    printf("grid barrier %3d CTAs: %.0f cycles (%.2f us)\n", grid, cyc / 10000.0, cyc / 10000.0 / 1965.0);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  const double ops = 148.0 * 1024 * K;
  auto timeit = [&](auto f) {
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  printf("random ld.cg 2MiB    : %.1f Gops/s\n", ops / 1e6 / timeit([&] { k_rand_ld<<<148, 1024>>>(bm, (1 << 19) - 1, 1, o2); }));
  printf("random red.or 2MiB   : %.1f Gops/s\n", ops / 1e6 / timeit([&] { k_rand_red<<<148, 1024>>>(bm, (1 << 19) - 1, 1); }));
  CK(cudaFuncSetAttribute(k_rand_red_shared, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  printf("random red.shared 160K: %.1f Gops/s\n",
         ops / 1e6 / timeit([&] { k_rand_red_shared<<<148, 1024, 160 * 1024>>>(o2, 1, 40 * 1024); }));
  printf("done: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
