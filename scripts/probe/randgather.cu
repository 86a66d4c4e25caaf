// randgather.cu -- probe: uniform random 4-byte gather rate vs loads in flight,
// array size and load flavour (measures the random-access roofline of B200 HBM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint64_t sm64(uint64_t x){ uint64_t z=x+0x9E3779B97F4A7C15ull; z=(z^(z>>30))*0xBF58476D1CE4E5B9ull; z=(z^(z>>27))*0x94D049BB133111EBull; return z^(z>>31);}
template<int ILP, int FL>
__global__ void __launch_bounds__(256) kg(const uint32_t* x, uint64_t len, uint64_t count, uint32_t* out){
  uint32_t acc=0; const uint64_t stride=(uint64_t)gridDim.x*blockDim.x;
  for(uint64_t i=(uint64_t)blockIdx.x*blockDim.x+threadIdx.x; i+(ILP-1)*stride<count; i+=ILP*stride){
    uint32_t t[ILP];
#pragma unroll
    for(int j=0;j<ILP;++j){ uint64_t r=sm64(i+j*stride); const uint32_t* p=x+(((r&0xFFFFFFFFull)*len)>>32);
      if(FL==0) t[j]=__ldcg(p); else if(FL==1) t[j]=__ldg(p); else { uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0,[%1];":"=r"(v):"l"(p)); t[j]=v; } }
#pragma unroll
    for(int j=0;j<ILP;++j) acc+=t[j];
  }
  if(acc==0x12345678) *out=acc;
}
template<int ILP,int FL> float run(const uint32_t* x,uint64_t len,uint64_t cnt,uint32_t* o,int grid){
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  kg<ILP,FL><<<grid,256>>>(x,len,cnt,o); cudaEventRecord(a); kg<ILP,FL><<<grid,256>>>(x,len,cnt,o); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms,a,b); return ms; }
int main(){
  int sms; cudaDeviceGetAttribute(&sms,cudaDevAttrMultiProcessorCount,0);
  uint64_t maxlen=1ull<<31; uint32_t* x; cudaMalloc(&x,maxlen*4); cudaMemset(x,1,maxlen*4); uint32_t* o; cudaMalloc(&o,4);
  uint64_t cnt=1ull<<28;
  for(uint64_t len: {1ull<<24, 1ull<<27, 1ull<<29, 1ull<<31}){
    for(int g: {sms*8, sms*32}){
      printf("len=%6llu MiB grid=%5d  ILP1 %.1f ILP2 %.1f ILP4 %.1f ILP8 %.1f ILP16 %.1f | ldg4 %.1f relaxed4 %.1f G/s\n",(unsigned long long)(len*4>>20),g,
        cnt/run<1,0>(x,len,cnt,o,g)/1e6, cnt/run<2,0>(x,len,cnt,o,g)/1e6, cnt/run<4,0>(x,len,cnt,o,g)/1e6, cnt/run<8,0>(x,len,cnt,o,g)/1e6, cnt/run<16,0>(x,len,cnt,o,g)/1e6,
        cnt/run<4,1>(x,len,cnt,o,g)/1e6, cnt/run<4,2>(x,len,cnt,o,g)/1e6);
    }
  }
  return 0;
}
