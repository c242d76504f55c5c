// Max co-resident clusters (cudaOccupancyMaxActiveClusters) of a 192-thread kernel at the GEMM's shared-memory sizes,
// for cluster sizes 1..16 (non-portable sizes enabled): can a split-K cluster of CS CTAs per n-tile be resident at once?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a cluster_occ.cu -o cluster_occ
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { if (p) p[0] = 1; }
int main() {
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int smem_kb : {100, 110, 200}) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
        for (int cs : {1, 2, 4, 5, 7, 8, 9, 10, 12, 14, 16}) {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(cs * 64);
            cfg.blockDim = dim3(192);
            cfg.dynamicSmemBytes = smem_kb * 1024;
            cudaLaunchAttribute at;
            at.id = cudaLaunchAttributeClusterDimension;
            at.val.clusterDim.x = cs;
            at.val.clusterDim.y = 1;
            at.val.clusterDim.z = 1;
            cfg.attrs = &at;
            cfg.numAttrs = 1;
            int n = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
            printf("smem %3d KB cluster %2d: max active clusters %4d (= %4d CTAs) %s\n", smem_kb, cs, n, n * cs,
                   cudaGetErrorString(e));
        }
    }
    return 0;
}
