// Microbenchmark: read-streaming bandwidth on B200 (one CTA per SM).
// A: LDG.128 grid-stride, U loads in flight per thread. B: TMA bulk-copy ring
// (1 producer thread, consumers wait full -> touch -> release), stage S bytes, N stages.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t sa(const void* p){return (uint32_t)__cvta_generic_to_shared(p);}
template<int U> __global__ void __launch_bounds__(1024,1) kA(const int4* __restrict__ p, int64_t n4, int* out){
  int acc=0; int64_t t=blockIdx.x*(int64_t)blockDim.x+threadIdx.x, st=(int64_t)gridDim.x*blockDim.x;
  for(int64_t i=t;i<n4;i+=st*U){
    int4 x[U];
#pragma unroll
    for(int u=0;u<U;++u){ int64_t j=i+u*st; x[u]= j<n4? __ldg(p+j):make_int4(0,0,0,0);}
#pragma unroll
    for(int u=0;u<U;++u) acc^=x[u].x^x[u].w;
  }
  if(acc==0x1234567) out[0]=acc;
}
__global__ void __launch_bounds__(544,1) kB(const char* __restrict__ p, int64_t bytes, int S, int N, int* out){
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[64], empty[64];
  int tid=threadIdx.x, warp=tid>>5, lane=tid&31;
  if(tid==0){ for(int b=0;b<N;++b){ asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;"::"r"(sa(&full[b]))); asm volatile("mbarrier.init.shared::cta.b64 [%0], 16;"::"r"(sa(&empty[b]))); } asm volatile("fence.mbarrier_init.release.cluster;":::"memory"); }
  __syncthreads();
  int64_t nch=bytes/S; int64_t my=(nch>blockIdx.x)?(nch-blockIdx.x+gridDim.x-1)/gridDim.x:0;
  int acc=0;
  if(warp==16){
    if(lane==0){
      for(int64_t i=0;i<my;++i){ int b=i%N; uint32_t ph=((i/N)&1)^1;
        asm volatile("{\n.reg .pred q;\nW1:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W1;\n}"::"r"(sa(&empty[b])),"r"(ph):"memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"::"r"(sa(&full[b])),"r"(S):"memory");
        const char* src=p+(blockIdx.x+i*gridDim.x)*(int64_t)S;
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"::"r"(sa(ring+(size_t)b*S)),"l"(src),"r"(S),"r"(sa(&full[b])):"memory");
      }
    }
  } else {
    for(int64_t i=0;i<my;++i){ int b=i%N; uint32_t ph=(i/N)&1;
      asm volatile("{\n.reg .pred q;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W2;\n}"::"r"(sa(&full[b])),"r"(ph):"memory");
      const int4* r=(const int4*)(ring+(size_t)b*S); int per=S/16/16;
      for(int k=0;k<per/32;++k){ int4 x=r[warp*per+k*32+lane]; acc^=x.x^x.w; }
      __syncwarp(); if(lane==0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];"::"r"(sa(&empty[b])):"memory");
    }
  }
  if(acc==0x1234567) out[0]=acc;
}
int main(){
  int64_t bytes=1536ll<<20; char* p; int* out; cudaMalloc(&p,bytes); cudaMalloc(&out,64); cudaMemset(p,1,bytes);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto timeit=[&](auto f){ f(); cudaDeviceSynchronize(); cudaEventRecord(a); for(int r=0;r<5;++r) f(); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b); return ms/5; };
  printf("A U=4: %.0f GB/s\n", bytes/1e6/timeit([&]{kA<4><<<148,1024>>>((const int4*)p,bytes/16,out);}));
  printf("A U=8: %.0f GB/s\n", bytes/1e6/timeit([&]{kA<8><<<148,1024>>>((const int4*)p,bytes/16,out);}));
  int cfg[][2]={{16384,4},{16384,5},{16384,8},{16384,12},{8192,8},{8192,16},{32768,4},{32768,6},{4096,16},{4096,32}};
  for(auto& c:cfg){ int S=c[0],N=c[1]; int sm=S*N; cudaFuncSetAttribute(kB,cudaFuncAttributeMaxDynamicSharedMemorySize,sm);
    float t=timeit([&]{kB<<<148,544,sm>>>(p,bytes,S,N,out);});
    printf("B S=%5d N=%2d (%3d KB): %.0f GB/s %s\n",S,N,sm/1024,bytes/1e6/t,cudaGetErrorString(cudaGetLastError())); }
  return 0;
}
