#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)
template<bool F64>
__global__ void vadd(const float4* __restrict__ w, const float4* __restrict__ y, const float4* __restrict__ z, float4* __restrict__ x, size_t n4){
  size_t stride = (size_t)gridDim.x*blockDim.x;
  for(size_t i = blockIdx.x*(size_t)blockDim.x + threadIdx.x; i < n4; i += 2*stride){
    float4 a0=__ldcs(w+i), b0=__ldcs(y+i), c0=__ldcs(z+i);
    bool has1 = i+stride<n4; float4 a1,b1,c1;
    if(has1){a1=__ldcs(w+i+stride); b1=__ldcs(y+i+stride); c1=__ldcs(z+i+stride);}
    float4 r0, r1;
    if(F64){
      r0.x=(float)(((double)a0.x+(double)b0.x)+(double)c0.x); r0.y=(float)(((double)a0.y+(double)b0.y)+(double)c0.y);
      r0.z=(float)(((double)a0.z+(double)b0.z)+(double)c0.z); r0.w=(float)(((double)a0.w+(double)b0.w)+(double)c0.w);
      r1.x=(float)(((double)a1.x+(double)b1.x)+(double)c1.x); r1.y=(float)(((double)a1.y+(double)b1.y)+(double)c1.y);
      r1.z=(float)(((double)a1.z+(double)b1.z)+(double)c1.z); r1.w=(float)(((double)a1.w+(double)b1.w)+(double)c1.w);
    } else {
      r0.x=a0.x+b0.x+c0.x; r0.y=a0.y+b0.y+c0.y; r0.z=a0.z+b0.z+c0.z; r0.w=a0.w+b0.w+c0.w;
      r1.x=a1.x+b1.x+c1.x; r1.y=a1.y+b1.y+c1.y; r1.z=a1.z+b1.z+c1.z; r1.w=a1.w+b1.w+c1.w;
    }
    __stcs(x+i, r0); if(has1) __stcs(x+i+stride, r1);
  }
}
__global__ void readsum(const float4* __restrict__ a, size_t n4, float* out){
  float s=0; size_t stride=(size_t)gridDim.x*blockDim.x;
  for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n4;i+=stride){float4 v=__ldcs(a+i); s+=v.x+v.y+v.z+v.w;}
  if(s==12345.f) out[0]=s;
}
__global__ void fill(float4* a, size_t n4){ size_t stride=(size_t)gridDim.x*blockDim.x; for(size_t i=blockIdx.x*(size_t)blockDim.x+threadIdx.x;i<n4;i+=stride) a[i]=make_float4(1,2,3,4);}
int main(){
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p,0));
  printf("name %s sms %d l2 %d smemOptin %zu smemPerSM %zu maxBlkSM %d regsSM %d mem %zu clock %d memclk %d busw %d coop %d\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor, p.maxBlocksPerMultiProcessor, p.regsPerMultiprocessor, p.totalGlobalMem, p.clockRate, p.memoryClockRate, p.memoryBusWidth, p.cooperativeLaunch);
  size_t n = 1ull<<28, n4=n/4;
  float4 *w,*y,*z,*x; CK(cudaMalloc(&w,n*4)); CK(cudaMalloc(&y,n*4)); CK(cudaMalloc(&z,n*4)); CK(cudaMalloc(&x,n*4));
  float* o; CK(cudaMalloc(&o,4));
  fill<<<1184,256>>>(w,n4); fill<<<1184,256>>>(y,n4); fill<<<1184,256>>>(z,n4);
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  int sms=p.multiProcessorCount;
  for(int occ : {4,8}) for(int f64=0; f64<2; ++f64){
    float best=1e9;
    for(int r=0;r<8;++r){ cudaEventRecord(a); if(f64) vadd<true><<<sms*occ,256>>>(w,y,z,x,n4); else vadd<false><<<sms*occ,256>>>(w,y,z,x,n4); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;}
    printf("vadd occ %d f64 %d: %.3f ms  %.1f GB/s\n", occ, f64, best, 16.0*n/best/1e6);
  }
  for(int occ: {4,8,16}){ float best=1e9; for(int r=0;r<8;++r){cudaEventRecord(a); readsum<<<sms*occ,256>>>(w,n4,o); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms,a,b); if(ms<best)best=ms;} printf("read occ %d: %.1f GB/s\n", occ, 4.0*n/best/1e6);}
  CK(cudaGetLastError());
  return 0;
}
