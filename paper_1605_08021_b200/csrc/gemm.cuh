// gemm.cuh -- FP64 DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA) tile machinery (K2).
//
// sm_100a has no fp64 kind for tcgen05.mma (ptxas: "Unknown modifier
// .kind::f64"), so the fp64 tensor path is the warp-level DMMA.  The projections
// Psi^T Y and Y - Psi C of the projector Q = I - Psi Psi^T
// are genuine dense contractions and run here.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace acp {

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// NN tile: C_tile(64 x 32) = A(64 x K) * B(K x 32); A col-major (lda), B col-major (ldb).
// 128 threads = 4 warps as 2 (m) x 2 (n); each warp owns 32 x 16 = 4 x 2 DMMA tiles.
// Epilogue functor interface (two phases, so that all global reads of a thread's 16 output
// elements are in flight together instead of serialising behind possibly-aliasing stores):
//   typename Ep::Regs;  ep.load(row, col, regs);  ep.store(row, col, acc, regs).
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
    // two halves of 8 elements each: loads of a half are all in flight together (~130 registers)
#pragma unroll
    for (int ih = 0; ih < 4; ih += 2) {
        typename Ep::Regs regs[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = m0 + wm * 32 + (ih + i) * 8 + g;
                    const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                    if (row < M && col < n) ep.load(row, col, regs[i][j][e]);
                }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = m0 + wm * 32 + (ih + i) * 8 + g;
                    const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                    if (row < M && col < n) ep.store(row, col, acc[ih + i][j][e], regs[i][j][e]);
                }
    }
}

// 32 x 32 NN tile with the epilogue operands PREFETCHED: every thread issues the global loads
// of its 8 output elements' epilogue operands before the K loop, so their latency overlaps the
// tile loads and the DMMA work (the PCG updates are bound by exactly those loads).  128 threads =
// 4 warps as 2 (m) x 2 (n), warp tile 16 x 16 = 2 x 2 DMMA tiles.
constexpr int NP_BM = 32, NP_BN = 32, NP_BK = 16;

template <class Ep>
__device__ __forceinline__ void nn_tile_pf(int M, int K, int n, const double* __restrict__ A, int lda,
                                           const double* __restrict__ B, int ldb, int m0, int n0, const Ep& ep) {
    __shared__ double As[NP_BK][NP_BM + 4];
    __shared__ double Bs[NP_BN][NP_BK + 4];
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    typename Ep::Regs regs[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 16 + i * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep.load(row, col, regs[i][j][e]);
            }
    double acc[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int k0 = 0; k0 < K; k0 += NP_BK) {
        for (int idx = tid; idx < NP_BK * NP_BM; idx += 128) {
            const int kk = idx / NP_BM, mm = idx % NP_BM;
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? A[(size_t)gk * lda + gm] : 0.0;
        }
        for (int idx = tid; idx < NP_BN * NP_BK; idx += 128) {
            const int nn = idx / NP_BK, kk = idx % NP_BK;
            const int gn = n0 + nn, gk = k0 + kk;
            Bs[nn][kk] = (gn < n && gk < K) ? B[(size_t)gn * ldb + gk] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < NP_BK; ks += 4) {
            double af[2], bf[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) af[i] = As[ks + t][wm * 16 + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = Bs[wn * 16 + j * 8 + g][ks + t];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 16 + i * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep.store(row, col, acc[i][j][e], regs[i][j][e]);
            }
}

// 64 x 64 NN tile for LARGE K (the PCG update at N_occ >= 64 and the SMW products are genuine
// FP64 GEMMs there): 256 threads = 8 warps as 2 (m) x 4 (n), warp tile 32 x 16 = 4 x 2 DMMA tiles,
// a GB_ST-stage cp.async ring of 32-deep K slices, then the two-phase epilogue.
constexpr int GB_BM = 64, GB_BN = 64, GB_BK = 32, GB_ST = 3, GB_LDA = GB_BM + 4, GB_LDB = GB_BK + 4;

template <int ST = GB_ST>
constexpr size_t nn_big_smem() { return (size_t)ST * (GB_BK * GB_LDA + GB_BN * GB_LDB) * sizeof(double); }

template <class Ep, int EPI = 0, int ST = GB_ST>
__device__ __forceinline__ void nn_tile_big(int M, int K, int n, const double* __restrict__ A, int lda,
                                            const double* __restrict__ B, int ldb, int m0, int n0, const Ep& ep) {
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;                              // [ST][GB_BK][GB_LDA]  (k-major: A(m, k) at [k][m])
    double* Bs = gsm + ST * GB_BK * GB_LDA;     // [ST][GB_BN][GB_LDB]  (B(k, n) at [n][k])
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    const int nk = (K + GB_BK - 1) / GB_BK;
    const bool vecA = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
    const bool vecB = ((ldb & 1) == 0) && ((((uintptr_t)B) & 15) == 0);
    auto load_stage = [&](int st, int k0) {
        double* as = As + st * GB_BK * GB_LDA;
        double* bs = Bs + st * GB_BN * GB_LDB;
        // A tile: GB_BK columns (k) of GB_BM contiguous rows (m)
        for (int c = tid; c < GB_BK * (GB_BM / 2); c += 256) {
            const int kk = c / (GB_BM / 2), mm = 2 * (c % (GB_BM / 2));
            const int gm = m0 + mm, gk = k0 + kk;
            if (vecA && gm + 1 < M && gk < K) {
                cp_async16(as + kk * GB_LDA + mm, A + (size_t)gk * lda + gm, true);
            } else {
                as[kk * GB_LDA + mm] = (gm < M && gk < K) ? A[(size_t)gk * lda + gm] : 0.0;
                as[kk * GB_LDA + mm + 1] = (gm + 1 < M && gk < K) ? A[(size_t)gk * lda + gm + 1] : 0.0;
            }
        }
        // B tile: GB_BN columns (n) of GB_BK contiguous k
        for (int c = tid; c < GB_BN * (GB_BK / 2); c += 256) {
            const int nn = c / (GB_BK / 2), kk = 2 * (c % (GB_BK / 2));
            const int gn = n0 + nn, gk = k0 + kk;
            if (vecB && gn < n && gk + 1 < K) {
                cp_async16(bs + nn * GB_LDB + kk, B + (size_t)gn * ldb + gk, true);
            } else {
                bs[nn * GB_LDB + kk] = (gn < n && gk < K) ? B[(size_t)gn * ldb + gk] : 0.0;
                bs[nn * GB_LDB + kk + 1] = (gn < n && gk + 1 < K) ? B[(size_t)gn * ldb + gk + 1] : 0.0;
            }
        }
    };
    double acc[4][2][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    // Epilogue order EPI: 0 = each half loaded then stored after the K loop (one half live),
    // 1 = both halves loaded after the K loop, 2 = the first half loaded before the K loop (its
    // operands do not depend on the product).  Selected per call site.
    typename Ep::Regs regs0[2][2][2];
    auto load_half0 = [&]() {
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int row = m0 + wm * 32 + i * 8 + g;
                    const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                    if (row < M && col < n) ep.load(row, col, regs0[i][j][e]);
                }
    };
    if constexpr (EPI == 2) load_half0();
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) {
        if (st < nk) load_stage(st, st * GB_BK);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        const int nxt = it + ST - 1;
        if (nxt < nk) load_stage(nxt % ST, nxt * GB_BK);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncthreads();
        const double* as = As + (it % ST) * GB_BK * GB_LDA;
        const double* bs = Bs + (it % ST) * GB_BN * GB_LDB;
#pragma unroll
        for (int ks = 0; ks < GB_BK; ks += 4) {
            double af[4], bf[2];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(ks + t) * GB_LDA + wm * 32 + i * 8 + g];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = bs[(wn * 16 + j * 8 + g) * GB_LDB + ks + t];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if constexpr (EPI == 0) {
        // one epilogue half live at a time (load, then store) keeps the registers in budget
#pragma unroll
        for (int ih = 0; ih < 4; ih += 2) {
            typename Ep::Regs regs[2][2][2];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = m0 + wm * 32 + (ih + i) * 8 + g;
                        const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                        if (row < M && col < n) ep.load(row, col, regs[i][j][e]);
                    }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int row = m0 + wm * 32 + (ih + i) * 8 + g;
                        const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                        if (row < M && col < n) ep.store(row, col, acc[ih + i][j][e], regs[i][j][e]);
                    }
        }
        return;
    }
    if constexpr (EPI == 1) load_half0();
    typename Ep::Regs regs1[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 32 + (2 + i) * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep.load(row, col, regs1[i][j][e]);
            }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 32 + i * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep.store(row, col, acc[i][j][e], regs0[i][j][e]);
            }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int row = m0 + wm * 32 + (2 + i) * 8 + g;
                const int col = n0 + wn * 16 + j * 8 + 2 * t + e;
                if (row < M && col < n) ep.store(row, col, acc[2 + i][j][e], regs1[i][j][e]);
            }
}

// 128 x 64 NN tile for the PCG update at N_occ >= 128 (configs[2], [4]: a genuine FP64 GEMM with
// K = N_occ): 256 threads = 8 warps as 4 (m) x 2 (n), warp tile 32 x 32 = 4 x 4 DMMA tiles (8 shared
// loads per 16 DMMAs instead of 6 per 8), XL_ST-stage cp.async ring of 16-deep K slices (27 KB per
// stage: two CTAs per SM), then the epilogue in four quarters of 8 elements per thread (each
// quarter's global loads in flight together).  A operand rows are 1.33x as long per byte of B as in
// the 64 x 64 tile, so the L2 -> SM operand stream per flop drops by a quarter.
constexpr int XL_BM = 128, XL_BN = 64, XL_BK = 16, XL_ST = 3, XL_LDA = XL_BM + 4, XL_LDB = XL_BK + 4;
constexpr int XL_GM = 16;   // m-tiles per rasterisation group

template <int ST = XL_ST>
constexpr size_t nn_xl_smem() { return (size_t)ST * (XL_BK * XL_LDA + XL_BN * XL_LDB) * sizeof(double); }

template <class Ep, int ST = XL_ST, bool SE = false>
__device__ __forceinline__ void nn_tile_xl(int M, int K, int n, const double* __restrict__ A, int lda,
                                           const double* __restrict__ B, int ldb, int m0, int n0, const Ep& ep) {
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;                            // [ST][XL_BK][XL_LDA]  A(m, k) at [k][m]
    double* Bs = gsm + ST * XL_BK * XL_LDA;      // [ST][XL_BN][XL_LDB]  B(k, n) at [n][k]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int nk = (K + XL_BK - 1) / XL_BK;
    const bool vecA = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0) && ((m0 & 1) == 0);
    const bool vecB = ((ldb & 1) == 0) && ((((uintptr_t)B) & 15) == 0);
    auto load_stage = [&](int st, int k0) {
        double* as = As + st * XL_BK * XL_LDA;
        double* bs = Bs + st * XL_BN * XL_LDB;
#pragma unroll
        for (int q = 0; q < (XL_BK * XL_BM / 2) / 256; ++q) {
            const int c = tid + q * 256;
            const int kk = c / (XL_BM / 2), mm = 2 * (c % (XL_BM / 2));
            const int gm = m0 + mm, gk = k0 + kk;
            if (vecA && gm + 1 < M && gk < K) {
                cp_async16(as + kk * XL_LDA + mm, A + (size_t)gk * lda + gm, true);
            } else {
                as[kk * XL_LDA + mm] = (gm < M && gk < K) ? A[(size_t)gk * lda + gm] : 0.0;
                as[kk * XL_LDA + mm + 1] = (gm + 1 < M && gk < K) ? A[(size_t)gk * lda + gm + 1] : 0.0;
            }
        }
#pragma unroll
        for (int q = 0; q < (XL_BN * XL_BK / 2) / 256; ++q) {
            const int c = tid + q * 256;
            const int nn = c / (XL_BK / 2), kk = 2 * (c % (XL_BK / 2));
            const int gn = n0 + nn, gk = k0 + kk;
            if (vecB && gn < n && gk + 1 < K) {
                cp_async16(bs + nn * XL_LDB + kk, B + (size_t)gn * ldb + gk, true);
            } else {
                bs[nn * XL_LDB + kk] = (gn < n && gk < K) ? B[(size_t)gn * ldb + gk] : 0.0;
                bs[nn * XL_LDB + kk + 1] = (gn < n && gk + 1 < K) ? B[(size_t)gn * ldb + gk + 1] : 0.0;
            }
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) {
        if (st < nk) load_stage(st, st * XL_BK);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        const int nxt = it + ST - 1;
        if (nxt < nk) load_stage(nxt % ST, nxt * XL_BK);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncthreads();
        const double* as = As + (it % ST) * XL_BK * XL_LDA + wm * 32 + g;
        const double* bs = Bs + (it % ST) * XL_BN * XL_LDB + (wn * 32 + g) * XL_LDB + t;
#pragma unroll
        for (int ks = 0; ks < XL_BK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[(ks + t) * XL_LDA + i * 8];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * XL_LDB + ks];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    if constexpr (SE) {
        // staged epilogue: the accumulators go through shared memory (the operand ring is free now),
        // then thread = row (coalesced 256-byte column segments per warp) with the 64 accumulator
        // registers released, so 16-32 elements' operand loads are in flight per thread
        __syncthreads();
        double* Cs = gsm;   // [XL_BN][XL_BM + 4]: 67.6 KB inside the 81 KB ring
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e)
                    Cs[(wn * 32 + j * 8 + 2 * t + e) * (XL_BM + 4) + wm * 32 + i * 8 + g] = acc[i][j][e];
        __syncthreads();
        const int r = tid % XL_BM, h = tid / XL_BM, row = m0 + r;
        constexpr int EC = sizeof(typename Ep::Regs) > 24 ? 8 : 16;
        for (int c0 = h * (XL_BN / 2); c0 < (h + 1) * (XL_BN / 2); c0 += EC) {
            typename Ep::Regs regs[EC];
#pragma unroll
            for (int c = 0; c < EC; ++c) {
                const int col = n0 + c0 + c;
                if (row < M && col < n) ep.load(row, col, regs[c]);
            }
#pragma unroll
            for (int c = 0; c < EC; ++c) {
                const int col = n0 + c0 + c;
                if (row < M && col < n) ep.store(row, col, Cs[(c0 + c) * (XL_BM + 4) + r], regs[c]);
            }
        }
        return;
    }
    // epilogue in chunks of EC elements per thread (all of a chunk's global loads in flight together)
    constexpr int EJ = sizeof(typename Ep::Regs) > 24 ? 2 : 4;   // j-columns per chunk
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + wm * 32 + i * 8 + g;
#pragma unroll
        for (int j0 = 0; j0 < 4; j0 += EJ) {
            typename Ep::Regs regs[EJ][2];
#pragma unroll
            for (int j = 0; j < EJ; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = n0 + wn * 32 + (j0 + j) * 8 + 2 * t + e;
                    if (row < M && col < n) ep.load(row, col, regs[j][e]);
                }
#pragma unroll
            for (int j = 0; j < EJ; ++j)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int col = n0 + wn * 32 + (j0 + j) * 8 + 2 * t + e;
                    if (row < M && col < n) ep.store(row, col, acc[i][j0 + j][e], regs[j][e]);
                }
        }
    }
}

// ---------------------------------------------------------------------------
// Warp-specialised persistent variant of the 128 x 64 tile (the PCG update for N_occ >= 64).
// The epilogue operands (2-4 streams of 8 B per output element) and the DMMA main loop used to run
// one after the other in every CTA (c4g: 5.9 ms per 4096 columns where the DMMA work alone is 3.7
// ms and the epilogue traffic 2.0 ms at HBM speed).  Here 8 COMPUTE warps run the main loop of tile
// i+1 while 8 EPILOGUE warps finish tile i: the compute warps park the 128 x 64 accumulator tile in
// shared memory and go on; the epilogue warps (thread = row, 8 columns per chunk, coalesced) load
// the operands, combine and store.  Hand-off by named barriers (FULL: accumulators written, EMPTY:
// read); the compute warps' own barrier is named too, so the two groups never wait on each other
// except at the hand-off.  One CTA per SM, tiles in m-fastest order (CTA b: tiles b, b + grid, ...).
constexpr int WS_CW = 8, WS_EW = 8, WS_T = 32 * (WS_CW + WS_EW), WS_LDC = XL_BM + 4;

template <int ST = XL_ST>
constexpr size_t nn_ws_smem() { return nn_xl_smem<ST>() + (size_t)XL_BN * WS_LDC * sizeof(double); }

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <class Ep, int ST = XL_ST>
__device__ __forceinline__ void nn_ws_persistent(int M, int K, int n, const double* __restrict__ A, int lda,
                                                 const double* __restrict__ B, int ldb, const Ep& ep) {
    extern __shared__ __align__(16) double gsm[];
    double* As = gsm;
    double* Bs = gsm + ST * XL_BK * XL_LDA;
    double* Cs = gsm + ST * (XL_BK * XL_LDA + XL_BN * XL_LDB);   // [XL_BN][WS_LDC]: acc(r, c) at [c][r]
    constexpr int BAR_FULL = 1, BAR_EMPTY = 2, BAR_MAIN = 3;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int mt = (M + XL_BM - 1) / XL_BM, nt = (n + XL_BN - 1) / XL_BN, ntiles = mt * nt;
    if (warp < WS_CW) {
        // ---------------- compute warps
        const int g = lane >> 2, t = lane & 3;
        const int wm = warp & 3, wn = warp >> 2;
        const int nk = (K + XL_BK - 1) / XL_BK;
        const bool vecA = ((lda & 1) == 0) && ((((uintptr_t)A) & 15) == 0);
        const bool vecB = ((ldb & 1) == 0) && ((((uintptr_t)B) & 15) == 0);
        bool first = true;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int m0 = (tile % mt) * XL_BM, n0 = (tile / mt) * XL_BN;
            int any = 0;
            for (int c = n0; c < min(n, n0 + XL_BN); ++c) any |= ep.active[c];
            if (!any) continue;   // the epilogue warps skip the same tiles
            auto load_stage = [&](int st, int k0) {
                double* as = As + st * XL_BK * XL_LDA;
                double* bs = Bs + st * XL_BN * XL_LDB;
#pragma unroll
                for (int q = 0; q < (XL_BK * XL_BM / 2) / 256; ++q) {
                    const int c = tid + q * 256;
                    const int kk = c / (XL_BM / 2), mm = 2 * (c % (XL_BM / 2));
                    const int gm = m0 + mm, gk = k0 + kk;
                    if (vecA && gm + 1 < M && gk < K) {
                        cp_async16(as + kk * XL_LDA + mm, A + (size_t)gk * lda + gm, true);
                    } else {
                        as[kk * XL_LDA + mm] = (gm < M && gk < K) ? A[(size_t)gk * lda + gm] : 0.0;
                        as[kk * XL_LDA + mm + 1] = (gm + 1 < M && gk < K) ? A[(size_t)gk * lda + gm + 1] : 0.0;
                    }
                }
#pragma unroll
                for (int q = 0; q < (XL_BN * XL_BK / 2) / 256; ++q) {
                    const int c = tid + q * 256;
                    const int nn = c / (XL_BK / 2), kk = 2 * (c % (XL_BK / 2));
                    const int gn = n0 + nn, gk = k0 + kk;
                    if (vecB && gn < n && gk + 1 < K) {
                        cp_async16(bs + nn * XL_LDB + kk, B + (size_t)gn * ldb + gk, true);
                    } else {
                        bs[nn * XL_LDB + kk] = (gn < n && gk < K) ? B[(size_t)gn * ldb + gk] : 0.0;
                        bs[nn * XL_LDB + kk + 1] = (gn < n && gk + 1 < K) ? B[(size_t)gn * ldb + gk + 1] : 0.0;
                    }
                }
            };
            double acc[4][4][2];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
            for (int st = 0; st < ST - 1; ++st) {
                if (st < nk) load_stage(st, st * XL_BK);
                cp_async_commit();
            }
            for (int it = 0; it < nk; ++it) {
                const int nxt = it + ST - 1;
                if (nxt < nk) load_stage(nxt % ST, nxt * XL_BK);
                cp_async_commit();
                cp_async_wait<ST - 1>();
                named_sync(BAR_MAIN, 32 * WS_CW);
                const double* as = As + (it % ST) * XL_BK * XL_LDA + wm * 32 + g;
                const double* bs = Bs + (it % ST) * XL_BN * XL_LDB + (wn * 32 + g) * XL_LDB + t;
#pragma unroll
                for (int ks = 0; ks < XL_BK; ks += 4) {
                    double af[4], bf[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) af[i] = as[(ks + t) * XL_LDA + i * 8];
#pragma unroll
                    for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * XL_LDB + ks];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
#pragma unroll
                        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
                }
                named_sync(BAR_MAIN, 32 * WS_CW);
            }
            cp_async_wait<0>();
            // hand the tile to the epilogue warps
            if (!first) named_sync(BAR_EMPTY, WS_T);
            first = false;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int e = 0; e < 2; ++e)
                        Cs[(wn * 32 + j * 8 + 2 * t + e) * WS_LDC + wm * 32 + i * 8 + g] = acc[i][j][e];
            __threadfence_block();
            named_arrive(BAR_FULL, WS_T);
        }
    } else {
        // ---------------- epilogue warps: thread e owns row m0 + (e % 128) of the tile and the
        // columns of half e / 128 (8 or 16 per chunk, all their loads in flight together)
        const int e = tid - 32 * WS_CW, r = e % XL_BM, ch = e / XL_BM;
        constexpr int NH = (32 * WS_EW) / XL_BM;                       // column groups
        constexpr int EC = sizeof(typename Ep::Regs) > 24 ? 8 : 16;   // columns per chunk
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int m0 = (tile % mt) * XL_BM, n0 = (tile / mt) * XL_BN;
            int any = 0;
            for (int c = n0; c < min(n, n0 + XL_BN); ++c) any |= ep.active[c];
            if (!any) continue;
            named_sync(BAR_FULL, WS_T);
            const int row = m0 + r;
            for (int c0 = ch * EC; c0 < XL_BN; c0 += NH * EC) {
                typename Ep::Regs regs[EC];
#pragma unroll
                for (int c = 0; c < EC; ++c) {
                    const int col = n0 + c0 + c;
                    if (row < M && col < n) ep.load(row, col, regs[c]);
                }
#pragma unroll
                for (int c = 0; c < EC; ++c) {
                    const int col = n0 + c0 + c;
                    if (row < M && col < n) ep.store(row, col, Cs[(c0 + c) * WS_LDC + r], regs[c]);
                }
            }
            named_arrive(BAR_EMPTY, WS_T);
        }
    }
}

// ---------------------------------------------------------------------------
// Split-K TN GEMM with the K-split reduced through distributed shared memory.
//   C(m x n, ld ldc) = alpha * A(:, m)^T B(:, n),  A: K x m (lda), B: K x n (ldb).
// One thread-block cluster of CS CTAs (cluster rank = K chunk) computes one BM x 32
// output tile; every CTA accumulates its K chunk with DMMA (cp.async double-buffered
// operand tiles), parks the partial tile in its shared memory, and after a cluster
// barrier each rank sums a slice of the tile over all CS ranks IN RANK ORDER through
// DSMEM.  No global partials, no atomics: the result depends only on (K, CS), not on n.
// `hook(col)` runs once per output column (rank 0, m-tile 0) after the tile is final.
constexpr int TC_BN = 32, TC_BK = 32, TC_PAD = 4, TC_ST = 4;  // TC_ST-stage cp.async ring

struct NoHook {
    __device__ __forceinline__ void operator()(int) const {}
    __device__ __forceinline__ bool tile_active(int, int) const { return true; }
    __device__ __forceinline__ bool tile_active_w(int, int, int) const { return true; }
};

template <int BM, int ST = TC_ST>
constexpr size_t tn_cluster_smem() {
    return (size_t)ST * (BM + TC_BN) * (TC_BK + TC_PAD) * sizeof(double);
}

template <int BM, class Hook, int ST = TC_ST>
__global__ void __launch_bounds__(128) k_tn_cluster(int K, int m, int n, const double* __restrict__ A, int lda,
                                                    const double* __restrict__ B, int ldb, int kchunk, double alpha,
                                                    double* __restrict__ C, int ldc, Hook hook) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double tsm[];
    constexpr int LD = TC_BK + TC_PAD;
    double* As = tsm;                         // [ST][BM][LD]
    double* Bs = tsm + ST * BM * LD;       // [ST][BN][LD]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 1, wn = warp >> 1;
    constexpr int WTM = BM / 2;               // warp tile rows (16 or 32)
    constexpr int TI = WTM / 8;               // DMMA tiles along m per warp
    const int CS = gridDim.x;
    const int rank = blockIdx.x;              // == cluster rank (cluster = (CS,1,1))
    // (walking the m-tiles of a column tile back to back, so its B slice is read from HBM once,
    // measured slower: c4g 4096 columns 4.95 vs 4.77 ms, 38088 columns 50.2 vs 46.9 ms)
    const int mt = gridDim.z;
    const int mtile = blockIdx.z;
    const int n0 = blockIdx.y * TC_BN, m0 = mtile * BM;
    pdl_wait();
    pdl_trigger();
    // Column tiles whose columns have all converged are skipped.  The decision must be uniform
    // over the cluster (a CTA that leaves early would strand its peers at the cluster barrier and
    // DSMEM reads).  With one m-tile (mt == 1) the only writer of the flags is this
    // cluster's own hook, which runs after the barrier below, so every rank reads the same
    // values.  With several m-tiles the hook of the z = 0 cluster may flip the flags while the
    // z > 0 clusters of the same column tile read them: there rank 0 decides and pushes its
    // decision to every peer before a cluster barrier.
    if (mt == 1) {
        if (!hook.tile_active(n0, n)) return;
    } else {
        __shared__ int s_act;
        if (rank == 0 && tid < CS) {
            const int act = hook.tile_active(n0, n) ? 1 : 0;
            *cluster.map_shared_rank(&s_act, tid) = act;
        }
        cluster.sync();
        if (!s_act) return;
    }
    const int kb = rank * kchunk;
    const int ke = min(K, kb + kchunk);
    const int nk = ke > kb ? (ke - kb + TC_BK - 1) / TC_BK : 0;

    auto load_stage = [&](int s, int k0) {
        double* as = As + s * BM * LD;
        double* bs = Bs + s * TC_BN * LD;
        for (int c = tid; c < BM * (TC_BK / 2); c += 128) {
            const int row = c / (TC_BK / 2), kk = 2 * (c % (TC_BK / 2));
            const int gm = m0 + row, gk = k0 + kk;
            const bool v = gm < m && gk < ke;
            cp_async16(as + row * LD + kk, v ? (const void*)(A + (size_t)gm * lda + gk) : (const void*)A, v);
        }
        for (int c = tid; c < TC_BN * (TC_BK / 2); c += 128) {
            const int col = c / (TC_BK / 2), kk = 2 * (c % (TC_BK / 2));
            const int gn = n0 + col, gk = k0 + kk;
            const bool v = gn < n && gk < ke;
            cp_async16(bs + col * LD + kk, v ? (const void*)(B + (size_t)gn * ldb + gk) : (const void*)B, v);
        }
    };

    double acc[TI][2][2];
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // ST-stage ring: ST - 1 stages in flight ahead of the one being multiplied (for the
    // 1D configs the whole K chunk, <= 160 rows, is requested at once: one memory latency)
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) {
        if (st < nk) load_stage(st, kb + st * TC_BK);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        const int nxt = it + ST - 1;
        if (nxt < nk) load_stage(nxt % ST, kb + nxt * TC_BK);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncthreads();
        const double* as = As + (it % ST) * BM * LD;
        const double* bs = Bs + (it % ST) * TC_BN * LD;
#pragma unroll
        for (int ks = 0; ks < TC_BK; ks += 4) {
            double af[TI], bf[2];
#pragma unroll
            for (int i = 0; i < TI; ++i) af[i] = as[(wm * WTM + i * 8 + g) * LD + ks + t];
#pragma unroll
            for (int j = 0; j < 2; ++j) bf[j] = bs[(wn * 16 + j * 8 + g) * LD + ks + t];
#pragma unroll
            for (int i = 0; i < TI; ++i)
#pragma unroll
                for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    // park the partial tile: Cs[row][col], row-major with LDC
    constexpr int LDC = TC_BN + 1;
    double* Cs = tsm;
#pragma unroll
    for (int i = 0; i < TI; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                Cs[(wm * WTM + i * 8 + g) * LDC + wn * 16 + j * 8 + 2 * t + e] = acc[i][j][e];
    cluster.sync();
    // rank r finalises elements e = r, r + CS, ... (column-major walk for coalesced stores)
    for (int e = rank * 128 + tid; e < BM * TC_BN; e += CS * 128) {
        const int row = e % BM, col = e / BM;
        // all CS remote loads in flight together (one DSMEM latency), then summed in rank order
        double part[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) part[q] = q < CS ? cluster.map_shared_rank(Cs, q)[row * LDC + col] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += part[q];
        const int gm = m0 + row, gn = n0 + col;
        if (gm < m && gn < n) C[(size_t)gn * ldc + gm] = alpha * s;
    }
    if (rank == 0 && mtile == 0 && tid < TC_BN && n0 + tid < n) hook(n0 + tid);
    cluster.sync();
}

// K split of the cluster projection: CS <= 8 ranks of kchunk rows (~160 per rank).  (Short K over
// up to 16 ranks, one memory latency per rank, measured slower on configs[1]: K2 17.5 vs 13.3 us.)
// 128 x 64 output tile of the split-K TN GEMM for m >= 128 (K2 at N_occ >= 128): 256 threads as
// 4 (m) x 2 (n) warps with 32 x 32 warp tiles (4 x 4 DMMA tiles: 8 shared loads per 16 DMMAs, the
// tile shape of the K3 main loop that reached 0.85 of the FP64 peak), 2-stage cp.async ring of
// 32-deep K slices (110 KB: two CTAs per SM), the same cluster split of K with the partial tiles
// reduced over the cluster in rank order through DSMEM, and the same per-column hook.
constexpr int TX_BM = 128, TX_BN = 64;
template <int BK, int ST>
constexpr size_t tn_xl_smem() { return (size_t)ST * (TX_BM + TX_BN) * (BK + TC_PAD) * sizeof(double); }

template <class Hook, int BK = 32, int ST = 2>
__global__ void __launch_bounds__(256, 2) k_tn_cluster_xl(int K, int m, int n, const double* __restrict__ A, int lda,
                                                          const double* __restrict__ B, int ldb, int kchunk,
                                                          double alpha, double* __restrict__ C, int ldc, Hook hook) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    extern __shared__ __align__(16) double tsm[];
    constexpr int LD = BK + TC_PAD;
    double* As = tsm;                           // [ST][TX_BM][LD]  A(k, m) at [m][k]
    double* Bs = tsm + ST * TX_BM * LD;         // [ST][TX_BN][LD]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const int CS = gridDim.x;
    const int rank = blockIdx.x;
    const int n0 = blockIdx.y * TX_BN, m0 = blockIdx.z * TX_BM;
    pdl_wait();
    pdl_trigger();
    // tile skipping decided uniformly per cluster (see k_tn_cluster)
    if (gridDim.z == 1) {
        if (!hook.tile_active_w(n0, n, TX_BN)) return;
    } else {
        __shared__ int s_act;
        if (rank == 0 && tid < CS) {
            const int act = hook.tile_active_w(n0, n, TX_BN) ? 1 : 0;
            *cluster.map_shared_rank(&s_act, tid) = act;
        }
        cluster.sync();
        if (!s_act) return;
    }
    const int kb = rank * kchunk;
    const int ke = min(K, kb + kchunk);
    const int nk = ke > kb ? (ke - kb + BK - 1) / BK : 0;
    auto load_stage = [&](int s, int k0) {
        double* as = As + s * TX_BM * LD;
        double* bs = Bs + s * TX_BN * LD;
#pragma unroll
        for (int q = 0; q < (TX_BM * (BK / 2)) / 256; ++q) {
            const int c = tid + q * 256;
            const int row = c / (BK / 2), kk = 2 * (c % (BK / 2));
            const int gm = m0 + row, gk = k0 + kk;
            const bool v = gm < m && gk < ke;
            cp_async16(as + row * LD + kk, v ? (const void*)(A + (size_t)gm * lda + gk) : (const void*)A, v);
        }
#pragma unroll
        for (int q = 0; q < (TX_BN * (BK / 2)) / 256; ++q) {
            const int c = tid + q * 256;
            const int col = c / (BK / 2), kk = 2 * (c % (BK / 2));
            const int gn = n0 + col, gk = k0 + kk;
            const bool v = gn < n && gk < ke;
            cp_async16(bs + col * LD + kk, v ? (const void*)(B + (size_t)gn * ldb + gk) : (const void*)B, v);
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
    for (int st = 0; st < ST - 1; ++st) {
        if (st < nk) load_stage(st, kb + st * BK);
        cp_async_commit();
    }
    for (int it = 0; it < nk; ++it) {
        const int nxt = it + ST - 1;
        if (nxt < nk) load_stage(nxt % ST, kb + nxt * BK);
        cp_async_commit();
        cp_async_wait<ST - 1>();
        __syncthreads();
        const double* as = As + (it % ST) * TX_BM * LD + (wm * 32 + g) * LD + t;
        const double* bs = Bs + (it % ST) * TX_BN * LD + (wn * 32 + g) * LD + t;
#pragma unroll
        for (int ks = 0; ks < BK; ks += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) af[i] = as[i * 8 * LD + ks];
#pragma unroll
            for (int j = 0; j < 4; ++j) bf[j] = bs[j * 8 * LD + ks];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    constexpr int LDC = TX_BN + 1;
    double* Cs = tsm;   // [TX_BM][LDC] (67 KB, inside the >= 92 KB ring)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e)
                Cs[(wm * 32 + i * 8 + g) * LDC + wn * 32 + j * 8 + 2 * t + e] = acc[i][j][e];
    cluster.sync();
    for (int e = rank * 256 + tid; e < TX_BM * TX_BN; e += CS * 256) {
        const int row = e % TX_BM, col = e / TX_BM;
        double part[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) part[q] = q < CS ? cluster.map_shared_rank(Cs, q)[row * LDC + col] : 0.0;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 16; ++q) s += part[q];
        const int gm = m0 + row, gn = n0 + col;
        if (gm < m && gn < n) C[(size_t)gn * ldc + gm] = alpha * s;
    }
    if (rank == 0 && blockIdx.z == 0 && tid < TX_BN && n0 + tid < n) hook(n0 + tid);
    cluster.sync();
}

inline bool tn_xl_on() {
    static const int v = getenv("ACP_K2_XL") ? atoi(getenv("ACP_K2_XL")) : 1;
    return v != 0;
}
inline void tn_split(int K, int& CS, int& kchunk) {
    CS = std::min(8, std::max(1, cdiv(K, 160)));
    kchunk = cdiv(cdiv(K, CS), TC_BK) * TC_BK;
    CS = cdiv(K, kchunk);
}

// Host launcher: returns false if the operand layout does not allow 16-byte cp.async.
template <class Hook>
bool launch_tn_cluster(acp_context* ctx, int K, int m, int n, double alpha, const double* A, int lda, const double* B,
                       int ldb, double* C, int ldc, Hook hook) {
    if ((K & 1) || (lda & 1) || (ldb & 1) || (((uintptr_t)A | (uintptr_t)B) & 15)) return false;
    int CS, kchunk;
    tn_split(K, CS, kchunk);
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(128, 1, 1);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = ctx->pdl ? 2 : 1;
    // the 32-row tile keeps the 4-stage ring (2 / 3 stages: 11.69 / 11.59 vs 11.57 ms/step on configs[1])
    if (m <= 32) {
        cfg.gridDim = dim3(CS, cdiv(n, TC_BN), cdiv(m, 32));
        cfg.dynamicSmemBytes = tn_cluster_smem<32>();
        func_attr((const void*)k_tn_cluster<32, Hook>, (int)tn_cluster_smem<32>(), true);
        ACP_CUDA(cudaLaunchKernelEx(&cfg, k_tn_cluster<32, Hook>, K, m, n, A, lda, B, ldb, kchunk, alpha, C, ldc, hook));
    } else if (m >= 256 && n >= 16384 && tn_xl_on()) {
        // c4g production widths (38088 / 46848 columns): 44.9 vs 47.6 ms per 38088 columns; at 4096
        // columns (5.26 vs 5.04 ms) and for N_occ = 128 (configs[2]: 0.513 vs 0.469 ms per 8192) the
        // 64 x 32 tile wins (more clusters for the SMs)
        cfg.blockDim = dim3(256, 1, 1);
        cfg.gridDim = dim3(CS, cdiv(n, TX_BN), cdiv(m, TX_BM));
        static const int v3 = getenv("ACP_K2_XL3") ? atoi(getenv("ACP_K2_XL3")) : 0;
        auto kern = v3 ? k_tn_cluster_xl<Hook, 16, 3> : k_tn_cluster_xl<Hook, 32, 2>;
        const size_t smem = v3 ? tn_xl_smem<16, 3>() : tn_xl_smem<32, 2>();
        cfg.dynamicSmemBytes = smem;
        func_attr((const void*)kern, (int)smem, true);
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, K, m, n, A, lda, B, ldb, kchunk, alpha, C, ldc, hook));
    } else {
        // 2-stage ring (55 KB -> up to 4 CTAs/SM instead of 2): K2 0.70 vs 0.52 of FP64 peak on
        // configs[2] (223 vs 241 ms/step), 0.78 vs 0.66 on configs[3] (745 vs 762) with 4 stages
        cfg.gridDim = dim3(CS, cdiv(n, TC_BN), cdiv(m, 64));
        cfg.dynamicSmemBytes = tn_cluster_smem<64, 2>();
        func_attr((const void*)k_tn_cluster<64, Hook, 2>, (int)tn_cluster_smem<64, 2>(), true);
        ACP_CUDA(cudaLaunchKernelEx(&cfg, k_tn_cluster<64, Hook, 2>, K, m, n, A, lda, B, ldb, kchunk, alpha, C, ldc,
                                    hook));
    }
    launched(ctx);
    return true;
}

}  // namespace acp
