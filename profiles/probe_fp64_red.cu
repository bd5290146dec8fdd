#include <cstdio>
#include <cuda_runtime.h>
__global__ void fma32(float* out, int iters){ float a=threadIdx.x*1e-3f,b=1.0001f,c=0.9999f,d=a+1,e=a+2,f=a+3,g=a+4,h=a+5;
 for(int i=0;i<iters;i++){ a=fmaf(a,b,c); d=fmaf(d,b,c); e=fmaf(e,b,c); f=fmaf(f,b,c); g=fmaf(g,b,c); h=fmaf(h,b,c);} out[blockIdx.x*blockDim.x+threadIdx.x]=a+d+e+f+g+h;}
__global__ void fma64(double* out, int iters){ double a=threadIdx.x*1e-3,b=1.0001,c=0.9999,d=a+1,e=a+2,f=a+3,g=a+4,h=a+5;
 for(int i=0;i<iters;i++){ a=fma(a,b,c); d=fma(d,b,c); e=fma(e,b,c); f=fma(f,b,c); g=fma(g,b,c); h=fma(h,b,c);} out[blockIdx.x*blockDim.x+threadIdx.x]=a+d+e+f+g+h;}
__global__ void red4(float4* buf, int n, int iters){ int t=blockIdx.x*blockDim.x+threadIdx.x; unsigned s=t*2654435761u;
 for(int i=0;i<iters;i++){ s=s*1664525u+1013904223u; float4* p=buf+(s%n);
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};"::"l"(p),"f"(1.f),"f"(1.f),"f"(1.f),"f"(1.f):"memory");}}
__global__ void red1(float* buf, int n, int iters){ int t=blockIdx.x*blockDim.x+threadIdx.x; unsigned s=t*2654435761u;
 for(int i=0;i<iters;i++){ s=s*1664525u+1013904223u; atomicAdd(buf+(s%n),1.f);}}
int main(){ float* o; cudaMalloc(&o, 1<<26); cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
 int blocks=148*8, th=256, it=4096;
 for(int r=0;r<2;r++){ cudaEventRecord(a); fma32<<<blocks,th>>>(o,it); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
 printf("fp32 fma: %.2f TFLOP/s\n", 2.0*6*it*(double)blocks*th/ms/1e9);
 for(int r=0;r<2;r++){ cudaEventRecord(a); fma64<<<blocks,th>>>((double*)o,it); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
 printf("fp64 fma: %.2f TFLOP/s\n", 2.0*6*it*(double)blocks*th/ms/1e9);
 int n=1<<22; it=256;
 for(int r=0;r<2;r++){ cudaEventRecord(a); red4<<<blocks,th>>>((float4*)o,n,it); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
 printf("red.v4 spread: %.1f G ops/s\n", (double)it*blocks*th/ms/1e6);
 for(int r=0;r<2;r++){ cudaEventRecord(a); red1<<<blocks,th>>>(o,n*4,it); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms,a,b);}
 printf("red.f32 spread: %.1f G ops/s\n", (double)it*blocks*th/ms/1e6);
 cudaDeviceProp p; cudaGetDeviceProperties(&p,0); printf("%s SMs=%d cc=%d.%d smemOptin=%zu l2=%d\n",p.name,p.multiProcessorCount,p.major,p.minor,p.sharedMemPerBlockOptin,p.l2CacheSize);
 printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));}
