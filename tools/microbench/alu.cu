// pipe-rate microbenchmark: FFMA, FMNMX, FSEL (+FSETP), mixed -- warp-instructions per cycle per SMSP
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kfmnmx(float* out, float s, int n){
  float a[8]; for(int j=0;j<8;j++) a[j]=threadIdx.x*0.001f+j;
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<8;j++){ float t; asm volatile("max.f32 %0, %1, %2;" : "=f"(t) : "f"(a[j]), "f"(s)); a[j]=t; }
  }
  float r=0; for(int j=0;j<8;j++) r+=a[j]; out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
__global__ void kfsel(float* out, float s, int n){
  float a[8]; for(int j=0;j<8;j++) a[j]=threadIdx.x*0.001f+j;
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<8;j++){ float t; asm volatile("{.reg .pred p; setp.ge.f32 p, %1, %2; selp.f32 %0, %1, %2, p;}" : "=f"(t) : "f"(a[j]), "f"(s)); a[j]=t; }
  }
  float r=0; for(int j=0;j<8;j++) r+=a[j]; out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
__global__ void kmix(float* out, float s, int n){
  float a[8], b[8]; for(int j=0;j<8;j++){ a[j]=threadIdx.x*0.001f+j; b[j]=a[j]*0.5f; }
  for (int k=0;k<n;k++){
#pragma unroll
    for(int j=0;j<8;j++){ float t; asm volatile("max.f32 %0, %1, %2;" : "=f"(t) : "f"(a[j]), "f"(s)); a[j]=t;
      float u; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(u) : "f"(b[j]), "f"(s), "f"(s)); b[j]=u; }
  }
  float r=0; for(int j=0;j<8;j++) r+=a[j]+b[j]; out[blockIdx.x*blockDim.x+threadIdx.x]=r;
}
int main(){
  float* o; cudaMalloc(&o, 148*8*256*4*4);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int n=20000; float ms; int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double slots = 148.0*4*clk*1e3;   // SMSP-cycles per second
  for(int rep=0;rep<2;rep++){
  double wi = 148.0*8*256/32*8*n;
  cudaEventRecord(e0); kfmnmx<<<148*8,256>>>(o,1.0001f,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("FMNMX: %.3f ms  %.2f warp-instr/cycle/SMSP\n", ms, wi/(ms*1e-3)/slots);
  cudaEventRecord(e0); kfsel<<<148*8,256>>>(o,1.0001f,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("FSETP+FSEL pairs: %.3f ms  %.2f pairs/cycle/SMSP\n", ms, wi/(ms*1e-3)/slots);
  cudaEventRecord(e0); kmix<<<148*8,256>>>(o,1.0001f,n); cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms,e0,e1);
  printf("FMNMX+FFMA pairs: %.3f ms  %.2f pairs/cycle/SMSP\n", ms, wi/(ms*1e-3)/slots);
  }
  return 0;
}
