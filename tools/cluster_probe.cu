// cluster_probe.cu -- how many thread-block clusters of size CL (2..16) a
// 544-thread CTA with ~192 KB of dynamic shared memory can keep co-resident
// on this GPU (cudaOccupancyMaxActiveClusters), i.e. how many SMs a
// cluster-per-row-band kernel can use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_probe tools/cluster_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void probe_kernel(float* p) {
  extern __shared__ float sm[];
  if (p) p[threadIdx.x] = sm[threadIdx.x];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smems[] = {3 * 65536 + 256, 3 * 58368 + 256, 2 * 65536 + 256};
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (size_t smem : smems) {
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int cl = 2; cl <= 16; ++cl) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cl;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.blockDim = dim3(544);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cfg.gridDim = dim3(cl * (sms / cl));
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
      printf("smem %6zu  cluster %2d: %3d clusters -> %3d SMs %s\n", smem, cl, n, n * cl,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
