// FP64 throughput on one B200: DMMA shapes (mma.sync .f64) and DFMA with ILP, whole chip.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
// Prints TF/s per variant (2 flops per FMA / per MMA multiply-add), timed with CUDA events
// over a persistent grid of 148 x BLK CTAs; every result feeds a store so nothing is elided.
#include <cstdio>

#define ITERS 4096

// DFMA, ILP independent chains per thread
template <int ILP>
__global__ void k_dfma(double* out, double b) {
    double a[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) a[i] = threadIdx.x * 1e-3 + i;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) a[i] = fma(a[i], b, 1e-9);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += a[i];
    if (s == 12345.0) out[blockIdx.x] = s;
}

// m8n8k4: A 1 reg, B 1 reg, C/D 2 regs per thread; ILP independent accumulators
template <int ILP>
__global__ void k_mma884(double* out, double b) {
    double a0 = threadIdx.x * 1e-3, b0 = b;
    double c[ILP][2];
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = i;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a0), "d"(b0));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[blockIdx.x] = s;
}

// m16n8k4: A 2 regs, B 1 reg, C/D 4 regs
template <int ILP>
__global__ void k_mma1684(double* out, double b) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, b0 = b;
    double c[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b0));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[blockIdx.x] = s;
}

// m16n8k8: A 4 regs, B 2 regs, C/D 4 regs
template <int ILP>
__global__ void k_mma1688(double* out, double b) {
    double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = b, b1 = b + 1;
    double c[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[blockIdx.x] = s;
}

// m16n8k16: A 8 regs, B 4 regs, C/D 4 regs
template <int ILP>
__global__ void k_mma16816(double* out, double b) {
    double a[8], bb[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) bb[i] = b + i;
    double c[ILP][4];
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = i;
    for (int k = 0; k < ITERS; ++k) {
#pragma unroll
        for (int i = 0; i < ILP; ++i)
            asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                         : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                         : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                           "d"(bb[0]), "d"(bb[1]), "d"(bb[2]), "d"(bb[3]));
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
    if (s == 12345.0) out[blockIdx.x] = s;
}

template <class K>
static void run(const char* name, K kern, int blk, int ctas_per_sm, double flops_per_thread_iter) {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 1 << 20);
    const int grid = nsm * ctas_per_sm;
    kern<<<grid, blk>>>(out, 1.0000001);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<<<grid, blk>>>(out, 1.0000001);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    const double fl = flops_per_thread_iter * (double)ITERS * blk * grid;
    printf("%-24s %4d thr x %d CTA/SM: %8.3f ms  %7.2f TF/s  (%s)\n", name, blk, ctas_per_sm, best, fl / best / 1e9,
           cudaGetErrorString(e));
    cudaFree(out);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
    // flops per THREAD per iteration: DFMA 2*ILP; an MMA m x n x k does 2mnk flops per warp
    run("dfma ilp4", k_dfma<4>, 256, 4, 2.0 * 4);
    run("dfma ilp8", k_dfma<8>, 256, 4, 2.0 * 8);
    run("dfma ilp8 1024thr", k_dfma<8>, 1024, 2, 2.0 * 8);
    run("mma m8n8k4 ilp4", k_mma884<4>, 256, 4, 2.0 * 8 * 8 * 4 * 4 / 32);
    run("mma m8n8k4 ilp8", k_mma884<8>, 256, 4, 2.0 * 8 * 8 * 4 * 8 / 32);
    run("mma m16n8k4 ilp4", k_mma1684<4>, 256, 4, 2.0 * 16 * 8 * 4 * 4 / 32);
    run("mma m16n8k8 ilp4", k_mma1688<4>, 256, 4, 2.0 * 16 * 8 * 8 * 4 / 32);
    run("mma m16n8k16 ilp2", k_mma16816<2>, 256, 4, 2.0 * 16 * 8 * 16 * 2 / 32);
    run("mma m16n8k16 ilp4", k_mma16816<4>, 256, 4, 2.0 * 16 * 8 * 16 * 4 / 32);
    return 0;
}
