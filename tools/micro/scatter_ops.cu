// Microbenchmark (dev): GPU-wide throughput of random scattered bit/byte
// updates, the cold-target step of the heavy-level sweep.
//   A red.global.or.b32 into a 2 MiB bitmap      B st.global.u8 into a 16 MiB byte map
//   C red.shared.or.b32 local (128 KB)           D red.shared::cluster.or.b32, partner CTA (cluster 2)
//   E st.global.b32 into 2 MiB (lossy baseline)
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t hsh(uint32_t x){ x^=x>>16; x*=0x7feb352dU; x^=x>>15; x*=0x846ca68bU; x^=x>>16; return x; }
constexpr int K = 256;
__global__ void __launch_bounds__(640) kA(uint32_t* bm, uint32_t mask_words, uint32_t seed){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  for(int k=0;k<K;++k){ uint32_t v=hsh(t*K+k+seed); asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;"::"l"(bm+((v>>5)&mask_words)),"r"(1u<<(v&31)):"memory"); }
}
__global__ void __launch_bounds__(640,1) kB(uint8_t* by, uint32_t mask, uint32_t seed){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  for(int k=0;k<K;++k){ uint32_t v=hsh(t*K+k+seed); asm volatile("st.global.u8 [%0], %1;"::"l"(by+(v&mask)),"h"((unsigned short)1):"memory"); }
}
__global__ void __launch_bounds__(640,1) kE(uint32_t* bm, uint32_t mask_words, uint32_t seed){
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  for(int k=0;k<K;++k){ uint32_t v=hsh(t*K+k+seed); asm volatile("st.global.b32 [%0], %1;"::"l"(bm+((v>>5)&mask_words)),"r"(1u<<(v&31)):"memory"); }
}
__global__ void __launch_bounds__(640,1) kC(uint32_t* out, uint32_t seed){
  extern __shared__ uint32_t s[];
  for(int i=threadIdx.x;i<32768;i+=blockDim.x) s[i]=0; __syncthreads();
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x; uint32_t base=(uint32_t)__cvta_generic_to_shared(s);
  for(int k=0;k<K*4;++k){ uint32_t v=hsh(t*K*4+k+seed); asm volatile("red.shared.or.b32 [%0], %1;"::"r"(base+((v>>5)&32767)*4),"r"(1u<<(v&31)):"memory"); }
  __syncthreads(); if(threadIdx.x==0) out[blockIdx.x]=s[seed&32767];
}
__global__ void __cluster_dims__(2,1,1) __launch_bounds__(640,1) kD(uint32_t* out, uint32_t seed){
  extern __shared__ uint32_t s[];
  for(int i=threadIdx.x;i<32768;i+=blockDim.x) s[i]=0;
  cg::cluster_group cl = cg::this_cluster(); cl.sync();
  uint32_t peer = cl.block_rank()^1;
  uint32_t base=(uint32_t)__cvta_generic_to_shared(s), rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;":"=r"(rb):"r"(base),"r"(peer));
  uint32_t t = blockIdx.x*blockDim.x+threadIdx.x;
  for(int k=0;k<K*4;++k){ uint32_t v=hsh(t*K*4+k+seed); asm volatile("red.shared::cluster.or.b32 [%0], %1;"::"r"(rb+((v>>5)&32767)*4),"r"(1u<<(v&31)):"memory"); }
  cl.sync(); if(threadIdx.x==0) out[blockIdx.x]=s[seed&32767];
}
int main(){
  uint32_t *bm; uint8_t* by; uint32_t* out; cudaMalloc(&bm,2<<20); cudaMalloc(&by,16<<20); cudaMalloc(&out,4096);
  cudaFuncSetAttribute(kC,cudaFuncAttributeMaxDynamicSharedMemorySize,131072);
  cudaFuncSetAttribute(kD,cudaFuncAttributeMaxDynamicSharedMemorySize,131072);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit=[&](auto f){ f(); cudaDeviceSynchronize(); cudaEventRecord(a); for(int r=0;r<5;++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); return ms/5; };
  double ops=148.0*640*K;
  printf("A red.global.or 2MiB : %.1f Gops/s\n", ops/1e6/timeit([&]{kA<<<148,640>>>(bm,(1<<19)-1,1);}));
  printf("A grid 74             : %.1f Gops/s\n", ops/2/1e6/timeit([&]{kA<<<74,640>>>(bm,(1<<19)-1,1);}));
  printf("A grid 37             : %.1f Gops/s\n", ops/4/1e6/timeit([&]{kA<<<37,640>>>(bm,(1<<19)-1,1);}));
  printf("A 148x128 thr         : %.1f Gops/s\n", ops/5/1e6/timeit([&]{kA<<<148,128>>>(bm,(1<<19)-1,1);}));
  printf("A 296x640 (2/SM)      : %.1f Gops/s\n", ops*2/1e6/timeit([&]{kA<<<296,640>>>(bm,(1<<19)-1,1);}));
  printf("A 16MiB region        : %.1f Gops/s\n", ops/1e6/timeit([&]{kA<<<148,640>>>((uint32_t*)by,(1<<22)-1,1);}));
  printf("B st.global.u8 16MiB : %.1f Gops/s\n", ops/1e6/timeit([&]{kB<<<148,640>>>(by,(16<<20)-1,1);}));
  printf("E st.global.b32 2MiB : %.1f Gops/s\n", ops/1e6/timeit([&]{kE<<<148,640>>>(bm,(1<<19)-1,1);}));
  printf("C red.shared local   : %.1f Gops/s\n", 4*ops/1e6/timeit([&]{kC<<<148,640,131072>>>(out,1);}));
  printf("D red.shared::cluster: %.1f Gops/s (%s)\n", 4*ops/1e6/timeit([&]{kD<<<148,640,131072>>>(out,1);}), cudaGetErrorString(cudaGetLastError()));
  return 0;
}
