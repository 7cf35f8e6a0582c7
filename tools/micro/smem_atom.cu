// Microbenchmark: random 32-bit shared-memory ops per SM (B200), 1024 threads/CTA, 1 CTA/SM.
// mode 0: LDS gather + xor; 1: red.shared.or (no return); 2: atom.shared.or with return;
// 3: LDS then conditional red (1/8 of lanes); 4: red.global.or to L2-resident 2 MiB bitmap (random)
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x){x^=x>>16;x*=0x7feb352dU;x^=x>>15;x*=0x846ca68bU;x^=x>>16;return x;}
template<int MODE>
__global__ void __launch_bounds__(1024,1) k(uint32_t* out, uint32_t* gbm, int iters, int words){
  extern __shared__ uint32_t s[];
  for(int i=threadIdx.x;i<words;i+=blockDim.x) s[i]=0;
  __syncthreads();
  uint32_t acc=0, x=hsh(threadIdx.x*7919u+blockIdx.x*104729u);
  for(int it=0;it<iters;++it){
#pragma unroll
    for(int j=0;j<8;++j){
      x = x*1664525u+1013904223u;
      uint32_t v = (x>>8) % (uint32_t)(words*32);
      uint32_t w = v>>5, b = 1u<<(v&31);
      if(MODE==0){ acc ^= s[w]; }
      else if(MODE==1){ asm volatile("red.shared.or.b32 [%0], %1;"::"r"((uint32_t)__cvta_generic_to_shared(s+w)),"r"(b):"memory"); }
      else if(MODE==2){ acc ^= atomicOr(s+w,b); }
      else if(MODE==3){ uint32_t o=s[w]; if(((o>>(v&31))&1u)==0 && (x&7)==0) atomicOr(s+w,b); acc^=o; }
      else if(MODE==4){ asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;"::"l"(gbm+(v&((1u<<19)-1))),"r"(b):"memory"); }
      else if(MODE==5){ acc ^= __ldcg(gbm+(x&((1u<<19)-1))); }
      else if(MODE==7){ asm volatile("st.global.u8 [%0], %1;"::"l"((unsigned char*)gbm+(v&((1u<<24)-1))),"r"(1u):"memory"); }
      else if(MODE==8){ asm volatile("st.global.u32 [%0], %1;"::"l"(gbm+(v&((1u<<22)-1))),"r"(b):"memory"); }
      else if(MODE==9){ asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;"::"l"(gbm+(v&((1u<<22)-1))),"r"(b):"memory"); }
      else if(MODE==6){ uint32_t r; asm volatile("atom.relaxed.gpu.global.or.b32 %0, [%1], %2;":"=r"(r):"l"(gbm+(v&((1u<<19)-1))),"r"(b):"memory"); acc^=r; }
    }
  }
  __syncthreads();
  if(threadIdx.x==0) out[blockIdx.x]=acc^s[0];
  else if(acc==0x12345) out[blockIdx.x]=acc;
}
int main(){
  int sms=148, words=36*1024, iters=200;
  uint32_t *out,*gbm; cudaMalloc(&out,4096*4); cudaMalloc(&gbm,(1<<22)*4); cudaMemset(gbm,0,(1<<22)*4);
  int smem=words*4;
  auto run=[&](auto kern,const char* name){
    cudaFuncSetAttribute(kern,cudaFuncAttributeMaxDynamicSharedMemorySize,smem);
    kern<<<sms,1024,smem>>>(out,gbm,iters,words); cudaDeviceSynchronize();
    cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for(int r=0;r<5;++r) kern<<<sms,1024,smem>>>(out,gbm,iters,words); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms,a,b); ms/=5;
    double ops=(double)sms*1024*iters*8;
    printf("%-28s %.3f ms  %.1f Gops/s  %.2f ops/clk/SM (1.965GHz)  err=%s\n",name,ms,ops/ms/1e6,ops/(ms*1e-3)/sms/1.965e9,cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0>,"LDS random");
  run(k<1>,"red.shared.or random");
  run(k<2>,"atom.shared.or ret random");
  run(k<3>,"LDS + 1/8 cond atom");
  run(k<4>,"red.global.or 2MiB random");
  run(k<5>,"ld.cg 2MiB random");
  run(k<6>,"atom.global.or ret 2MiB random");
  run(k<7>,"st.u8 16MiB random");
  run(k<8>,"st.u32 16MiB random");
  run(k<9>,"red.or 16MiB random");
  return 0;
}
