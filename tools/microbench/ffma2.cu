#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2(u64 a, u64 b, u64 c){ u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__global__ void kscalar(float* out, float s, int n){
  float a[8]; for(int j=0;j<8;j++) a[j]=threadIdx.x*0.001f+j;
  float b = s, c = s*0.5f;
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<8;j++) a[j]=__fmaf_rn(a[j], b, c);
  }
  float r=0; for(int j=0;j<8;j++) r+=a[j]; out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
__global__ void kpair(float* out, float s, int n){
  u64 a[4]; for(int j=0;j<4;j++){ float x=threadIdx.x*0.001f+j, y=x+1; asm("mov.b64 %0, {%1,%2};" : "=l"(a[j]) : "f"(x), "f"(y)); }
  u64 b, c; float c0 = s*0.5f; asm("mov.b64 %0, {%1,%2};" : "=l"(b) : "f"(s), "f"(s)); asm("mov.b64 %0, {%1,%2};" : "=l"(c) : "f"(c0), "f"(c0));
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<4;j++) a[j]=f2(a[j], b, c);
  }
  float r=0; for(int j=0;j<4;j++){ float x,y; asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[j])); r+=x+y;} out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
__global__ void kmufu(float* out, float s, int n){
  float a[8]; for(int j=0;j<8;j++) a[j]=-(threadIdx.x*0.001f+j)*1e-3f;
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<8;j++){ float e; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a[j])); a[j]=e*-1e-3f; }
  }
  float r=0; for(int j=0;j<8;j++) r+=a[j]; out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*256*4*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n=20000; float ms;
  for(int rep=0;rep<2;rep++){
  cudaEventRecord(e0); kscalar<<<148*8,256>>>(o,1.0001f,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  double flops = 148.0*8*256*8*n; printf("scalar FFMA: %.3f ms, %.2f T fma/s\n", ms, flops/ms/1e9);
  cudaEventRecord(e0); kpair<<<148*8,256>>>(o,1.0001f,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("FFMA2      : %.3f ms, %.2f T fma/s (lane-ops)\n", ms, flops/ms/1e9);
  cudaEventRecord(e0); kmufu<<<148*8,256>>>(o,1.0001f,n/4); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("MUFU ex2   : %.3f ms, %.2f T ex2/s\n", ms, flops/4/ms/1e9);
  }
  return 0;
}
