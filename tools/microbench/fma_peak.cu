// Microbenchmark: FP32 FFMA vs FFMA2 throughput, smem LDS.64 throughput, pinned H2D bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void ffma_k(float* out, float a, float b, int iters){
  float acc[16];
  #pragma unroll
  for(int i=0;i<16;i++) acc[i]=threadIdx.x*1e-3f+i;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++) acc[i]=fmaf(acc[i],a,b);
  }
  float s=0; for(int i=0;i<16;i++) s+=acc[i];
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c){
  unsigned long long r; 
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)), "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__global__ void ffma2_k(float* out, float a, float b, int iters){
  float2 acc[16];
  #pragma unroll
  for(int i=0;i<16;i++) acc[i]=make_float2(threadIdx.x*1e-3f+i, i*0.5f);
  float2 A=make_float2(a,a*0.5f), B=make_float2(b,b*2.f);
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++) acc[i]=ffma2(acc[i],A,B);
  }
  float s=0; for(int i=0;i<16;i++) s+=acc[i].x+acc[i].y;
  out[blockIdx.x*blockDim.x+threadIdx.x]=s;
}
__global__ void lds_k(float* out, int iters){
  __shared__ float2 sm[2048];
  for(int i=threadIdx.x;i<2048;i+=blockDim.x) sm[i]=make_float2(i,i);
  __syncthreads();
  float2 acc=make_float2(0,0);
  int base=threadIdx.x&1023;
  for(int it=0; it<iters; ++it){
    #pragma unroll
    for(int i=0;i<16;i++){ float2 v=sm[(base+i*32+it)&2047]; acc.x+=v.x; acc.y+=v.y; }
  }
  out[blockIdx.x*blockDim.x+threadIdx.x]=acc.x+acc.y;
}
int main(){
  int dev=0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,dev));
  printf("{\"gpu\":\"%s\",\"sms\":%d,\"clock_khz\":%d}\n", p.name, p.multiProcessorCount, p.clockRate);
  float* out; CK(cudaMalloc(&out, 148*8*256*sizeof(float)*4));
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grid=p.multiProcessorCount*4, block=256, iters=20000;
  for(int rep=0;rep<2;rep++){
    ffma_k<<<grid,block>>>(out,1.0001f,0.999f,iters); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); ffma_k<<<grid,block>>>(out,1.0001f,0.999f,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double fl=2.0*16*iters*(double)grid*block; printf("{\"ffma_tflops\":%.2f}\n", fl/ms/1e9);
    ffma2_k<<<grid,block>>>(out,1.0001f,0.999f,iters); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); ffma2_k<<<grid,block>>>(out,1.0001f,0.999f,iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    fl=4.0*16*iters*(double)grid*block; printf("{\"ffma2_tflops\":%.2f}\n", fl/ms/1e9);
    lds_k<<<grid,block>>>(out,iters/4); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); lds_k<<<grid,block>>>(out,iters/4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms,e0,e1);
    double by=8.0*16*(iters/4)*(double)grid*block; printf("{\"lds64_TBps\":%.2f, \"B_per_clk_per_sm\":%.1f}\n", by/ms/1e9, by/(ms*1e-3)/p.multiProcessorCount/(p.clockRate*1e3));
  }
  // pinned H2D
  size_t nb=256ull<<20; void* h; void* d; CK(cudaMallocHost(&h,nb)); CK(cudaMalloc(&d,nb));
  memset(h,0,nb);
  for(int rep=0;rep<3;rep++){
    cudaEventRecord(e0); CK(cudaMemcpyAsync(d,h,nb,cudaMemcpyHostToDevice)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("{\"h2d_pinned_GBps\":%.1f}\n", nb/ms/1e6);
  }
  void* hp=malloc(nb); memset(hp,1,nb);
  for(int rep=0;rep<2;rep++){
    cudaEventRecord(e0); CK(cudaMemcpy(d,hp,nb,cudaMemcpyHostToDevice)); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms,e0,e1); printf("{\"h2d_pageable_GBps\":%.1f}\n", nb/ms/1e6);
  }
  return 0;
}
