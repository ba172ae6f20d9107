// gemm.cuh -- FP64 DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA) tile machinery (K2).
//
// sm_100a has no fp64 kind for tcgen05.mma (ptxas: "Unknown modifier
// .kind::f64"), so the fp64 tensor path is the warp-level DMMA.  The projections
// Psi^T Y and Y - Psi C of the projector Q = I - Psi Psi^T
// are genuine dense contractions and run here.
#pragma once

#include "common.cuh"

namespace acp {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// NN tile: C_tile(64 x 32) = A(64 x K) * B(K x 32); A col-major (lda), B col-major (ldb).
// 128 threads = 4 warps as 2 (m) x 2 (n); each warp owns 32 x 16 = 4 x 2 DMMA tiles.
// The epilogue functor is called as ep(row, col, acc) for every in-range element.
constexpr int NN_BM = 64, NN_BN = 32, NN_BK = 16;

template <class Ep>
__device__ __forceinline__ void nn_tile(int M, int K, int n, const double* __restrict__ A, int lda,
                                        const double* __restrict__ B, int ldb, int m0, int n0, Ep& ep) {
    __shared__ double As[NN_BK][NN_BM + 4];
    __shared__ double Bs[NN_BN][NN_BK + 4];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int k0 = 0; k0 < K; k0 += NN_BK) {
        // A tile: BK x BM, m contiguous in global (col-major)
        for (int idx = tid; idx < NN_BK * NN_BM; idx += 128) {
            const int kk = idx / NN_BM, mm = idx % NN_BM;
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gk * lda + gm] : 0.0;
        }
        // B tile: BN x BK, k contiguous in global
        for (int idx = tid; idx < NN_BN * NN_BK; idx += 128) {
            const int nn = idx / NN_BK, kk = idx % NN_BK;
            const int gn = n0 + nn, gk = k0 + kk;
            Bs[nn][kk] = (gn < n && gk < K) ? B[(size_t)gn * ldb + gk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < NN_BK; ks += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = As[ks + t][wm * 32 + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = Bs[wn * 16 + j * 8 + g][ks + t];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 32 + i * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep(row, col, acc[i][j][e]);
            }
}

}  // namespace acp
