// Microbenchmarks calibrating single-SM latencies on B200 (smem double loads, DFMA chains,
// __syncthreads with 1024 threads, cluster barriers).  Standalone: nvcc -arch=sm_100a mb.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void k_smem_fma(long long* out, int iters, int sync_every) {
    __shared__ double s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 1.0 + i * 1e-6;
    __syncthreads();
    double acc = 0.0;
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) {
        acc += s[(threadIdx.x + 32 * k) & 4095] * s[(threadIdx.x * 3 + k) & 4095];
        if (sync_every && (k % sync_every) == 0) __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = t1 - t0; }
    if (acc == 12345.0) out[1] = 1;
}

__global__ void k_dfma_chain(long long* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0000001;
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) a = fma(a, b, 1e-9);
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    if (a == 12345.0) out[1] = 1;
}

__global__ void k_sync(long long* out, int iters) {
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
}

__global__ void k_cluster_sync(long long* out, int iters) {
    cg::cluster_group cl = cg::this_cluster();
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) cl.sync();
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    long long h[2];
    const int it = 4096;
    int ths[] = {32, 256, 1024};
    for (int T : ths) {
        k_smem_fma<<<1, T>>>(d, it, 0);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("smem-load+dfma loop, %4d threads: %.1f cycles/iter\n", T, (double)h[0] / it);
        k_smem_fma<<<1, T>>>(d, it, 8);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("  + __syncthreads every 8 iters: %.1f cycles/iter\n", (double)h[0] / it);
        k_dfma_chain<<<1, T>>>(d, it);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("dependent DFMA chain,  %4d threads: %.1f cycles/fma\n", T, (double)h[0] / it);
        k_sync<<<1, T>>>(d, it);
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("__syncthreads,         %4d threads: %.1f cycles\n", T, (double)h[0] / it);
    }
    for (int cs : {2, 8, 16}) {
        cudaFuncSetAttribute(k_cluster_sync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cs); cfg.blockDim = dim3(1024);
        cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
        a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
        cfg.attrs = a; cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_cluster_sync, d, it);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
        printf("cluster.sync, %2d CTAs x 1024: %.1f cycles (%s)\n", cs, (double)h[0] / it, cudaGetErrorString(e));
    }
    return 0;
}
