// Max co-resident clusters for a 160-thread kernel at a given dynamic smem, per cluster size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dummy(int *p) { extern __shared__ int s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
    int smems[] = {100 * 1024, 160 * 1024, 200 * 1024, 227 * 1024};
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int sm : smems)
        for (int cs : {1, 2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(128);
            cfg.blockDim = dim3(160);
            cfg.dynamicSmemBytes = sm;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            int nc = -1;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&nc, k_dummy, &cfg);
            printf("smem %6d KB cluster %2d: max active clusters %4d -> CTAs %4d (%s)\n", sm / 1024, cs, nc, nc * cs,
                   cudaGetErrorString(e));
        }
    return 0;
}
