// dense.cu -- small dense fp64 kernels kept on the device: LU solve (SMW core of
// Eq. dyson4), cyclic Jacobi symmetric eigensolver (phonon modes
// D u = omega^2 u; Rayleigh-Ritz in the ground state) and Cholesky.
// All run in ONE CTA (the matrices are O(N_e) x O(N_e) and off the bandwidth-
// critical loop); reductions use fixed orders, so results are deterministic.
#include "common.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace acp {

__device__ __forceinline__ void block_argmax_abs(double val, int idx, double* sv, int* si, double& best, int& bi) {
    // lowest index among maximal |val|
    for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, val, o);
        int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov > val || (ov == val && oi < idx)) {
            val = ov;
            idx = oi;
        }
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) {
        sv[w] = val;
        si[w] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = -1.0;
        int ii = 1 << 30;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i)
            if (sv[i] > b || (sv[i] == b && si[i] < ii)) {
                b = sv[i];
                ii = si[i];
            }
        sv[0] = b;
        si[0] = ii;
    }
    __syncthreads();
    best = sv[0];
    bi = si[0];
    __syncthreads();
}

// Blocked LU with partial pivoting of A (n x n col-major) applied to B (n x nrhs), then back
// substitution -- the SMW core solve of Eq. dyson4.  One CTA of 1024 threads; A
// (and B when both fit) in shared memory.  Panels of LU_NB = 32 columns:
//   1. warp 0 factors the panel alone (pivot = first row of maximal |a| in the column, LAPACK
//      idamax rule; row swaps inside the panel; multipliers; rank-1 updates) with warp-level
//      synchronisation only;
//   2. the panel's row swaps are applied, in order, to every other column of [A | B];
//   3. U12 = L11^{-1} A12 (unit lower triangular solve, one warp per column);
//   4. A22 -= L21 U12 (threads over 4-row segments, K = LU_NB);
// then a warp-per-right-hand-side back substitution with U (no block barriers: the columns of
// B are independent).  ~4 block barriers per panel instead of ~3 per column.
constexpr int LU_NB = 32;
__global__ void __launch_bounds__(1024) k_lu_solve(double* __restrict__ Ag, int n, double* __restrict__ Bg, int nrhs,
                                                   int use_smem, int* __restrict__ status, int accumulate) {
    // use_smem: 0 = both in global memory, 1 = A in shared memory, 2 = A and B in shared memory
    extern __shared__ double lsm[];
    __shared__ int s_piv[LU_NB];
    __shared__ int s_sing;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31, nwarp = nt >> 5;
    double* A = Ag;
    double* B = Bg;
    if (use_smem >= 1) {
        A = lsm;
        for (long long e = tid; e < (long long)n * n; e += nt) A[e] = Ag[e];
    }
    if (use_smem >= 2) {
        B = lsm + (size_t)n * n;
        for (long long e = tid; e < (long long)n * nrhs; e += nt) B[e] = Bg[e];
    }
    if (tid == 0) s_sing = 0;
    __syncthreads();
    auto col = [&](int j) -> double* { return j < n ? A + (size_t)j * n : B + (size_t)(j - n) * n; };
    const int ntot = n + nrhs;
    for (int p0 = 0; p0 < n; p0 += LU_NB) {
        const int pw = min(LU_NB, n - p0);
        // ---- 1. panel factorisation by warp 0
        if (warp == 0) {
            for (int kk = 0; kk < pw; ++kk) {
                const int k = p0 + kk;
                double* ck = A + (size_t)k * n;
                double bv = -1.0;
                int bi = 1 << 30;
                for (int i = k + lane; i < n; i += 32) {
                    const double a = fabs(ck[i]);
                    if (a > bv) {
                        bv = a;
                        bi = i;
                    }
                }
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                    if (ov > bv || (ov == bv && oi < bi)) {
                        bv = ov;
                        bi = oi;
                    }
                }
                // singular column: flag it and continue branch-free (the result is discarded)
                if (bv == 0.0) {
                    bi = k;
                    if (lane == 0) s_sing = 1;
                }
                if (lane == 0) s_piv[kk] = bi;
                if (bi != k && lane < pw) {  // swap rows k and bi inside the panel
                    double* cj = A + (size_t)(p0 + lane) * n;
                    const double t = cj[k];
                    cj[k] = cj[bi];
                    cj[bi] = t;
                }
                __syncwarp();
                const double rp = bv == 0.0 ? 0.0 : 1.0 / ck[k];
                for (int i = k + 1 + lane; i < n; i += 32) ck[i] *= rp;
                __syncwarp();
                for (int jj = kk + 1; jj < pw; ++jj) {
                    double* cj = A + (size_t)(p0 + jj) * n;
                    const double akj = cj[k];
                    for (int i = k + 1 + lane; i < n; i += 32) cj[i] -= ck[i] * akj;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        if (s_sing) {
            if (tid == 0) *status = 1;
            return;
        }
        // ---- 2. apply the panel's row swaps (in order) to the other columns of [A | B]
        for (int j = tid; j < ntot; j += nt) {
            if (j >= p0 && j < p0 + pw) continue;
            double* cj = col(j);
            for (int kk = 0; kk < pw; ++kk) {
                const int k = p0 + kk, pr = s_piv[kk];
                if (pr != k) {
                    const double t = cj[k];
                    cj[k] = cj[pr];
                    cj[pr] = t;
                }
            }
        }
        __syncthreads();
        const int r0 = p0 + pw;  // first row / column of the trailing block
        if (r0 >= ntot) break;
        // ---- 3. U12 = L11^{-1} A12 for the trailing columns of [A | B] (warp per column)
        for (int j = r0 + warp; j < ntot; j += nwarp) {
            double* cj = col(j);
            for (int kk = 0; kk < pw; ++kk) {
                const int k = p0 + kk;
                const double xk = cj[k];
                const int i = k + 1 + lane;
                if (i < r0) cj[i] -= A[(size_t)k * n + i] * xk;
                __syncwarp();
            }
        }
        __syncthreads();
        // ---- 4. A22 -= L21 U12 (rows r0..n-1), threads over 4-row segments of each column
        const int rows = n - r0;
        if (rows > 0) {
            const int segs = (rows + 3) >> 2;
            const int cols = ntot - r0;
            for (int e = tid; e < segs * cols; e += nt) {
                const int jj = e / segs, sg = e - jj * segs;
                double* cj = col(r0 + jj);
                const int i0 = r0 + 4 * sg;
                double acc[4] = {0.0, 0.0, 0.0, 0.0};
                for (int kk = 0; kk < pw; ++kk) {
                    const double u = cj[p0 + kk];
                    const double* lk = A + (size_t)(p0 + kk) * n;
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (i0 + t < n) acc[t] += lk[i0 + t] * u;
                }
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (i0 + t < n) cj[i0 + t] -= acc[t];
            }
        }
        __syncthreads();
    }
    // ---- back substitution U X = B: one warp per right-hand side, no block barriers
    for (int j = warp; j < nrhs; j += nwarp) {
        double* bj = B + (size_t)j * n;
        for (int k = n - 1; k >= 0; --k) {
            const double x = bj[k] / A[(size_t)k * n + k];
            __syncwarp();
            if (lane == 0) bj[k] = x;
            for (int i = lane; i < k; i += 32) bj[i] -= A[(size_t)k * n + i] * x;
            __syncwarp();
        }
    }
    __syncthreads();
    if (use_smem >= 2)
        for (long long e = tid; e < (long long)n * nrhs; e += nt) Bg[e] = B[e];
    if (tid == 0 && !accumulate) *status = 0;
}

// ---------------------------------------------------------------------------
// Multi-kernel blocked LU for the SMW core (any n): the matrix [A | B] is ONE column-major
// n x (n + nrhs) array (ld n).  Per panel of pw <= 32 columns:
//   k_lu_panel   one CTA factors the panel (rows p0..n-1), in shared memory when it fits:
//                block-wide first-max pivot search, row swap inside the panel, then a
//                row-parallel elimination (thread per row: l_i = a_ik / a_kk once, then the
//                row's remaining panel entries) -- 3 barriers per column;
//   k_lu_swap    applies the panel's row interchanges, in order, to every other column;
//   k_lu_trsm12  U12 = L11^{-1} A12 (unit lower, one warp per column, shuffles);
//   gemm_nn      A22 -= L21 U12 on the DMMA tensor path (the O(n^3) part, whole GPU).
// Back substitution by 32-row blocks from the bottom: k_lu_bsub (warp per right-hand side)
// then gemm_nn for the rows above.
__global__ void __launch_bounds__(1024) k_lu_panel(double* __restrict__ AB, int n, int p0, int pw, int use_smem,
                                                   int* __restrict__ piv, int* __restrict__ status) {
    extern __shared__ double psm[];
    __shared__ double red_v[32];
    __shared__ int red_i[32];
    __shared__ int s_p;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), nwarp = nt >> 5;
    const int R = n - p0;                      // panel rows
    double* P = use_smem ? psm : AB + (size_t)p0 * n + p0;
    const int ld = use_smem ? R : n;
    if (use_smem) {
        for (int e = tid; e < R * pw; e += nt) {
            const int jj = e / R, i = e - jj * R;
            P[(size_t)jj * R + i] = AB[(size_t)(p0 + jj) * n + p0 + i];
        }
        __syncthreads();
    }
    for (int kk = 0; kk < pw; ++kk) {
        double* ck = P + (size_t)kk * ld;
        double bv = -1.0;
        int bi = 1 << 30;
        for (int i = kk + tid; i < R; i += nt) {
            const double a = fabs(ck[i]);
            if (a > bv) {
                bv = a;
                bi = i;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
        }
        __syncthreads();
        if (warp == 0) {
            bv = lane < nwarp ? red_v[lane] : -1.0;
            bi = lane < nwarp ? red_i[lane] : (1 << 30);
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) {
                s_p = bv == 0.0 ? -1 : bi;
                piv[p0 + kk] = p0 + (bv == 0.0 ? kk : bi);
                if (bv == 0.0) *status = 1;
            }
        }
        __syncthreads();
        const int pr = s_p < 0 ? kk : s_p;
        if (pr != kk)
            for (int jj = tid; jj < pw; jj += nt) {
                double* cj = P + (size_t)jj * ld;
                const double t = cj[kk];
                cj[kk] = cj[pr];
                cj[pr] = t;
            }
        __syncthreads();
        const double akk = ck[kk];
        const double rp = akk == 0.0 ? 0.0 : 1.0 / akk;
        for (int i = kk + 1 + tid; i < R; i += nt) ck[i] *= rp;
        __syncthreads();
        // rank-1 update of the panel's remaining columns: warps over columns, lanes over rows
        for (int jj = kk + 1 + warp; jj < pw; jj += nwarp) {
            double* cj = P + (size_t)jj * ld;
            const double akj = cj[kk];
            for (int i = kk + 1 + lane; i < R; i += 32) cj[i] -= ck[i] * akj;
        }
        __syncthreads();
    }
    if (use_smem)
        for (int e = tid; e < R * pw; e += nt) {
            const int jj = e / R, i = e - jj * R;
            AB[(size_t)(p0 + jj) * n + p0 + i] = P[(size_t)jj * R + i];
        }
}

__global__ void k_lu_swap(double* __restrict__ AB, int n, int ntot, int p0, int pw, const int* __restrict__ piv) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= ntot || (j >= p0 && j < p0 + pw)) return;
    double* cj = AB + (size_t)j * n;
    for (int kk = 0; kk < pw; ++kk) {
        const int k = p0 + kk, pr = piv[k];
        if (pr != k) {
            const double t = cj[k];
            cj[k] = cj[pr];
            cj[pr] = t;
        }
    }
}

// U12 = L11^{-1} A12 for columns j >= p0 + pw: one warp per column, lane i holds row p0 + i;
// the unit lower triangle L11 (pw x pw) is staged in shared memory once per CTA.
__global__ void __launch_bounds__(256) k_lu_trsm12(double* __restrict__ AB, int n, int ntot, int p0, int pw) {
    __shared__ double Ls[32][33];
    for (int e = threadIdx.x; e < pw * pw; e += blockDim.x) {
        const int k = e / pw, i = e - k * pw;
        Ls[k][i] = AB[(size_t)(p0 + k) * n + p0 + i];
    }
    __syncthreads();
    const int w = blockIdx.x * (blockDim.x >> 5) + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    const int j = p0 + pw + w;
    if (j >= ntot) return;
    double* cj = AB + (size_t)j * n + p0;
    double x = lane < pw ? cj[lane] : 0.0;
    for (int k = 0; k < pw; ++k) {
        const double xk = __shfl_sync(0xffffffffu, x, k);
        if (lane > k && lane < pw) x -= Ls[k][lane] * xk;
    }
    if (lane < pw) cj[lane] = x;
}

// X_b = U_bb^{-1} B_b for the rows [q0, q0 + qb) (qb <= 32): one warp per right-hand side, the
// diagonal block of U staged in shared memory with reciprocal diagonal.
__global__ void __launch_bounds__(256) k_lu_bsub(double* __restrict__ AB, int n, int nrhs, int q0, int qb,
                                                 int r0) {
    __shared__ double Us[32][33];
    __shared__ double rd[32];
    for (int e = threadIdx.x; e < qb * qb; e += blockDim.x) {
        const int k = e / qb, i = e - k * qb;
        Us[k][i] = AB[(size_t)(q0 + k) * n + q0 + i];
    }
    __syncthreads();
    if (threadIdx.x < qb) rd[threadIdx.x] = 1.0 / Us[threadIdx.x][threadIdx.x];
    __syncthreads();
    const int w = blockIdx.x * (blockDim.x >> 5) + __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
    const int lane = threadIdx.x & 31;
    if (w >= nrhs) return;
    double* bj = AB + (size_t)(n + r0 + w) * n + q0;
    double x = lane < qb ? bj[lane] : 0.0;
    for (int k = qb - 1; k >= 0; --k) {
        const double xk = __shfl_sync(0xffffffffu, x, k) * rd[k];
        if (lane == k) x = xk;
        if (lane < k) x -= Us[k][lane] * xk;
    }
    if (lane < qb) bj[lane] = x;
}

// U X = B in place for upper-triangular U (first n columns of AB, n x (n + nrhs), ld n): 32-row
// blocks from the bottom, k_lu_bsub (warp per right-hand side) + DMMA gemm_nn for the rows above.
void upper_solve_blocked(acp_context* ctx, double* AB, int n, int nrhs) {
    for (int q1 = n; q1 > 0; q1 -= 32) {
        const int q0 = std::max(0, q1 - 32);
        for (int r0 = 0; r0 < nrhs; r0 += 65535 * 8) {  // grid.x limit
            const int nr = std::min(nrhs - r0, 65535 * 8);
            k_lu_bsub<<<cdiv((long long)nr * 32, 256), 256, 0, ctx->stream>>>(AB, n, nr, q0, q1 - q0, r0);
            launched(ctx);
        }
        if (q0 > 0)
            gemm_nn(ctx, q0, q1 - q0, nrhs, -1.0, AB + (size_t)q0 * n, n, AB + (size_t)n * n + q0, n, 1.0,
                    AB + (size_t)n * n, n);
    }
}

// Solve A X = B in place; AB is n x (n + nrhs) column-major ([A | B], ld n).

void lu_solve_blocked(acp_context* ctx, double* AB, int n, int nrhs) {
    const int ntot = n + nrhs;
    int* piv = ctx->wsi("lu_piv", n);
    // deferred mode (acp_dyson): the status accumulates in the device statistics, read at the end
    int* st = ctx->defer ? reinterpret_cast<int*>(ctx->defer_stats + 6) : ctx->wsi("lu_status", 1);
    if (!ctx->defer) ACP_CUDA(cudaMemsetAsync(st, 0, sizeof(int), ctx->stream));
    func_attr((const void*)k_lu_panel, 200 * 1024);
    for (int p0 = 0; p0 < n; p0 += 32) {
        const int pw = std::min(32, n - p0);
        const int R = n - p0;
        const size_t pbytes = (size_t)R * pw * sizeof(double);
        const int use_smem = pbytes <= 200 * 1024;
        {
            const int T = R <= 512 ? 256 : 1024;  // fewer warps -> cheaper barriers on short panels
            k_lu_panel<<<1, T, use_smem ? pbytes : 0, ctx->stream>>>(AB, n, p0, pw, use_smem, piv, st);
        }
        launched(ctx);
        k_lu_swap<<<cdiv(ntot, 128), 128, 0, ctx->stream>>>(AB, n, ntot, p0, pw, piv);
        launched(ctx);
        const int r0 = p0 + pw;
        if (r0 >= ntot) continue;
        k_lu_trsm12<<<cdiv((long long)(ntot - r0) * 32, 256), 256, 0, ctx->stream>>>(AB, n, ntot, p0, pw);
        launched(ctx);
        if (r0 < n)
            gemm_nn(ctx, n - r0, pw, ntot - r0, -1.0, AB + (size_t)p0 * n + r0, n, AB + (size_t)r0 * n + p0, n, 1.0,
                    AB + (size_t)r0 * n + r0, n);
    }
    upper_solve_blocked(ctx, AB, n, nrhs);
    if (ctx->defer) return;
    int* hp = static_cast<int*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, st, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    if (*hp != 0) throw Error(ACP_ERR_SINGULAR, "singular SMW core in blocked LU (n = " + std::to_string(n) + ")");
}

void lu_solve(acp_context* ctx, double* A, int n, double* B, int nrhs) {
    // deferred mode (acp_dyson): the status accumulates in the device statistics
    int* st = ctx->defer ? reinterpret_cast<int*>(ctx->defer_stats + 6) : ctx->wsi("lu_status", 1);
    const size_t abytes = (size_t)n * n * sizeof(double), bbytes = (size_t)n * nrhs * sizeof(double);
    const int use_smem = abytes + bbytes <= 224 * 1024 ? 2 : abytes <= 224 * 1024 ? 1 : 0;
    const size_t bytes = use_smem == 2 ? abytes + bbytes : use_smem == 1 ? abytes : 0;
    func_attr((const void*)k_lu_solve, 224 * 1024);
    k_lu_solve<<<1, 1024, bytes, ctx->stream>>>(A, n, B, nrhs, use_smem, st, ctx->defer);
    launched(ctx);
    if (ctx->defer) return;
    int* hp = static_cast<int*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, st, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    const int h = *hp;
    if (h != 0) throw Error(ACP_ERR_SINGULAR, "singular matrix in LU solve (n = " + std::to_string(n) + ")");
}

// Parallel cyclic Jacobi (round-robin "circle" ordering): A (n x n col-major, symmetric) ->
// eigenvalues w (ascending), eigenvectors V (n x n col-major) if V != nullptr.  One CTA; A in
// shared memory when it fits.  Round r of a sweep (m = n rounded up to even, index m-1 a dummy
// when n is odd) rotates the disjoint pairs (r, m-1) and ((r+k) mod (m-1), (r-k) mod (m-1)),
// k = 1..m/2-1 -- all pairs once per sweep, pair indices computed, not shuffled.  Rotations with
// |a_pq| <= 1e-300 or |a_pq| below rounding of the diagonal are skipped; sweeps stop when the
// off-diagonal Frobenius norm is <= 1e-14 of the total (eigenvalue error second order in it).
__global__ void __launch_bounds__(1024) k_jacobi(double* __restrict__ Ag, int n, double* __restrict__ V,
                                                 double* __restrict__ w, int* __restrict__ order,
                                                 double* __restrict__ rot, int max_sweeps, int use_smem) {
    extern __shared__ double jsm[];
    __shared__ double red[2][32];
    __shared__ int s_done;
    const int tid = threadIdx.x, nt = blockDim.x;
    double* A = Ag;
    if (use_smem) {
        A = jsm;
        for (long long e = tid; e < (long long)n * n; e += nt) A[e] = Ag[e];
    }
    const int m = (n % 2) ? n + 1 : n;
    const int np = m / 2;
    if (V)
        for (long long e = tid; e < (long long)n * n; e += nt) V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
    __syncthreads();
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double off = 0.0, tot = 0.0;
        for (int j = tid >> 5; j < n; j += nt >> 5)
            for (int i = tid & 31; i < n; i += 32) {
                const double a = A[(size_t)j * n + i];
                tot += a * a;
                if (i != j) off += a * a;
            }
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            tot += __shfl_xor_sync(0xffffffffu, tot, o);
        }
        if ((tid & 31) == 0) {
            red[0][tid >> 5] = off;
            red[1][tid >> 5] = tot;
        }
        __syncthreads();
        if (tid == 0) {
            double so = 0.0, st = 0.0;
            for (int i = 0; i < nt / 32; ++i) {
                so += red[0][i];
                st += red[1][i];
            }
            s_done = (so <= 1e-28 * st) ? 1 : 0;
        }
        __syncthreads();
        if (s_done) break;
        for (int r = 0; r < m - 1; ++r) {
            for (int k = tid; k < np; k += nt) {
                int p, q;
                if (k == 0) {
                    p = r;
                    q = m - 1;
                } else {
                    p = (r + k) % (m - 1);
                    q = (r - k + (m - 1)) % (m - 1);
                }
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, sn = 0.0;
                if (q < n) {
                    const double apq = A[(size_t)q * n + p];
                    const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
                    if (fabs(apq) > 1e-300 && fabs(apq) > 1e-18 * (fabs(app) + fabs(aqq))) {
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        sn = t * c;
                    }
                }
                rot[4 * k] = c;
                rot[4 * k + 1] = sn;
                rot[4 * k + 2] = p;
                rot[4 * k + 3] = q;
            }
            __syncthreads();
            // columns: A <- A J (and V <- V J); threads over (pair, row)
            for (int k = tid >> 5; k < np; k += nt >> 5) {
                const double sn = rot[4 * k + 1];
                const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
                if (sn == 0.0 || q >= n) continue;
                const double c = rot[4 * k];
                for (int i = tid & 31; i < n; i += 32) {
                const double aip = A[(size_t)p * n + i], aiq = A[(size_t)q * n + i];
                A[(size_t)p * n + i] = c * aip - sn * aiq;
                A[(size_t)q * n + i] = sn * aip + c * aiq;
                if (V) {
                    const double vip = V[(size_t)p * n + i], viq = V[(size_t)q * n + i];
                    V[(size_t)p * n + i] = c * vip - sn * viq;
                    V[(size_t)q * n + i] = sn * vip + c * viq;
                }
                }
            }
            __syncthreads();
            // rows: A <- J^T A; threads over (pair, column)
            for (int k = tid >> 5; k < np; k += nt >> 5) {
                const double sn = rot[4 * k + 1];
                const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
                if (sn == 0.0 || q >= n) continue;
                const double c = rot[4 * k];
                for (int j = tid & 31; j < n; j += 32) {
                    const double apj = A[(size_t)j * n + p], aqj = A[(size_t)j * n + q];
                    A[(size_t)j * n + p] = c * apj - sn * aqj;
                    A[(size_t)j * n + q] = sn * apj + c * aqj;
                }
            }
            __syncthreads();
        }
    }
    // sort eigenvalues ascending (selection by rank, stable on ties by index)
    for (int i = tid; i < n; i += nt) {
        const double di = A[(size_t)i * n + i];
        int rank = 0;
        for (int j = 0; j < n; ++j) {
            const double dj = A[(size_t)j * n + j];
            if (dj < di || (dj == di && j < i)) ++rank;
        }
        w[rank] = di;
        order[rank] = i;
    }
}

__global__ void k_permute_cols(int n, const double* __restrict__ Vin, const int* __restrict__ order,
                               double* __restrict__ Vout) {
    long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= (long long)n * n) return;
    const int i = (int)(e % n), j = (int)(e / n);
    Vout[e] = Vin[(size_t)order[j] * n + i];
}

// Eigenvalues only, n <= 32: cyclic Jacobi inside ONE warp with the matrix in registers (lane l
// holds column l), no block barriers.  Round r of a sweep rotates the disjoint pairs of the circle
// ordering (m = 32 slots, slots >= n are dummies); lane l learns its partner and the pair's
// rotation by shuffles, updates its column (rows p, q) locally and combines with its partner's
// column for the column rotation.  Sweeps stop when the off-diagonal Frobenius norm is
// <= 1e-14 of the total (same criterion as k_jacobi).  Ascending sort by rank at the end.
__global__ void __launch_bounds__(32) k_jacobi_warp(const double* __restrict__ Ag, int n, double* __restrict__ w,
                                                    int max_sweeps) {
    const int l = threadIdx.x;
    double a[32];  // a[i] = A(i, l)
#pragma unroll
    for (int i = 0; i < 32; ++i) a[i] = (l < n && i < n) ? Ag[(size_t)l * n + i] : (i == l ? 1.0 : 0.0) * 0.0;
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        double off = 0.0, tot = 0.0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
            tot += a[i] * a[i];
            if (i != l) off += a[i] * a[i];
        }
        for (int o = 16; o > 0; o >>= 1) {
            off += __shfl_xor_sync(0xffffffffu, off, o);
            tot += __shfl_xor_sync(0xffffffffu, tot, o);
        }
        if (off <= 1e-28 * tot) break;
        for (int r = 0; r < 31; ++r) {
            // partner of slot l in round r of the circle method on 32 slots (slot 31 fixed)
            int q;
            if (l == 31) q = r;
            else if (l == r) q = 31;
            else q = ((2 * r - l) % 31 + 31) % 31;
            const int p = min(l, q), qq = max(l, q);
            // a_pp, a_qq, a_pq from the owners: lane p holds column p (a_pp = a[p], a_pq = a[qq])
            double app = 0.0, aqq = 0.0, apq = 0.0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (i == l) app = a[i];          // diagonal of my column
                if (i == q) apq = a[i];          // A(q, l)
            }
            aqq = __shfl_sync(0xffffffffu, app, q);
            // my diagonal is app (column l); rotation angle from the pair (p, qq)
            const double dpp = l == p ? app : aqq, dqq = l == p ? aqq : app;
            double c = 1.0, sn = 0.0;
            if (qq < n && fabs(apq) > 1e-300 && fabs(apq) > 1e-18 * (fabs(dpp) + fabs(dqq))) {
                const double th = (dqq - dpp) / (2.0 * apq);
                const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                c = 1.0 / sqrt(t * t + 1.0);
                sn = t * c;
            }
            // the pair's rotation is the one computed by its lower lane p (rounding could make the
            // two lanes' copies of a_pq differ slightly)
            c = __shfl_sync(0xffffffffu, c, p);
            sn = __shfl_sync(0xffffffffu, sn, p);
            // column rotation: A <- A J; column p' = c col_p - s col_q, column q' = s col_p + c col_q
            const double sgn = l == p ? -1.0 : 1.0;  // p: c*mine - s*partner ; q: c*mine + s*partner
            double partner[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) partner[i] = __shfl_sync(0xffffffffu, a[i], q);
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = c * a[i] + sgn * sn * partner[i];
            // row rotation: A <- J^T A on rows (p_k, q_k) of every pair k, in my column.  The pair
            // of row i is (i, partner(i)) with the rotation owned by lanes i / partner(i).
#pragma unroll
            for (int i = 0; i < 32; ++i) partner[i] = a[i];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                int qi;
                if (i == 31) qi = r;
                else if (i == r) qi = 31;
                else qi = ((2 * r - i) % 31 + 31) % 31;
                const double ci = __shfl_sync(0xffffffffu, c, i);   // (c, s) already uniform per pair
                const double si = __shfl_sync(0xffffffffu, sn, i);
                const double sg = i < qi ? -1.0 : 1.0;
                a[i] = ci * partner[i] + sg * si * partner[qi];
            }
        }
    }
    // eigenvalues: diagonal entries, sorted ascending by rank (stable by index)
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (i == l) d = a[i];
    int rank = 0;
    for (int j = 0; j < n; ++j) {
        const double dj = __shfl_sync(0xffffffffu, d, j);
        if (dj < d || (dj == d && j < l)) ++rank;
    }
    if (l < n) w[rank] = d;
}

// ---------------------------------------------------------------------------------------------
// Eigenvalues only (the phonon spectrum lambda of D): Householder reduction to
// tridiagonal form, then Sturm-count multisection.  Block Jacobi needs O(n^3) work per sweep and
// ~10 sweeps; this is one O(4n^3/3) reduction plus an O(n^2) eigenvalue search.
//
// k_tridiag<GRID>: lower Householder tridiagonalisation of the full symmetric column-major A.
// Step k: x = A(k+1:, k); beta = -sign(x0) ||x||; v = [1, x(1:)/(x0-beta)]; tau = (beta-x0)/beta;
// p = tau A22 v; w = p - (tau/2)(p.v) v; A22 -= v w^T + w v^T.  Every CTA derives v (and w) itself
// from the same data with the same fixed-order reduction, so the copies agree bitwise and only the
// matvec and the rank-2 update are distributed (one warp per column).  GRID=false: one CTA, A in
// shared memory, __syncthreads; GRID=true: cooperative grid over A in global memory, grid.sync().
template <bool GRID>
__global__ void __launch_bounds__(1024) k_tridiag(double* __restrict__ Ag, int n, double* __restrict__ pg,
                                                   double* __restrict__ dout, double* __restrict__ eout) {
    namespace cg = cooperative_groups;
    extern __shared__ double tsm[];
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    double* vs = tsm;           // n
    double* ws = vs + n;        // n
    double* red = ws + n;       // 32
    double* A = GRID ? Ag : red + 32;
    if (!GRID) {
        for (int i = tid; i < n * n; i += nt) A[i] = Ag[i];
        __syncthreads();
    }
    const int gw = GRID ? blockIdx.x * nw + warp : warp;  // global warp id
    const int tw = GRID ? gridDim.x * nw : nw;            // total warps
    auto gsync = [&]() {
        if (GRID) {
            __threadfence();
            cg::this_grid().sync();
        } else {
            __syncthreads();
        }
    };
    // fixed-order block sum (same result in every CTA)
    auto bsum = [&](double a) {
#pragma unroll
        for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
        __syncthreads();
        if (lane == 0) red[warp] = a;
        __syncthreads();
        double t = 0.0;
        for (int q = 0; q < nw; ++q) t += red[q];
        return t;
    };
    for (int k = 0; k + 2 < n; ++k) {
        const int m = n - k - 1;
        const double* x = A + (size_t)k * n + k + 1;
        const double x0 = x[0];
        double part = 0.0;
        for (int i = 1 + tid; i < m; i += nt) part += x[i] * x[i];
        const double xn2 = bsum(part);
        if (GRID ? blockIdx.x == 0 && tid == 0 : tid == 0) dout[k] = A[(size_t)k * n + k];
        if (xn2 == 0.0) {  // already reduced: tau = 0, no update
            if (GRID ? blockIdx.x == 0 && tid == 0 : tid == 0) eout[k] = x0;
            gsync();
            continue;
        }
        const double beta = x0 >= 0.0 ? -sqrt(x0 * x0 + xn2) : sqrt(x0 * x0 + xn2);
        const double tau = (beta - x0) / beta;
        const double sc = 1.0 / (x0 - beta);
        for (int i = tid; i < m; i += nt) vs[i] = i == 0 ? 1.0 : x[i] * sc;
        __syncthreads();
        // p_i = tau * A22(:, i) . v   (A22 symmetric: column i, contiguous)
        for (int i = gw; i < m; i += tw) {
            const double* col = A + (size_t)(k + 1 + i) * n + k + 1;
            double a = 0.0;
            for (int j = lane; j < m; j += 32) a += col[j] * vs[j];
#pragma unroll
            for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (lane == 0) pg[i] = tau * a;
        }
        gsync();
        if (GRID ? blockIdx.x == 0 && tid == 0 : tid == 0) eout[k] = beta;
        part = 0.0;
        for (int i = tid; i < m; i += nt) part += pg[i] * vs[i];
        const double K = 0.5 * tau * bsum(part);
        for (int i = tid; i < m; i += nt) ws[i] = pg[i] - K * vs[i];
        __syncthreads();
        for (int j = gw; j < m; j += tw) {
            double* col = A + (size_t)(k + 1 + j) * n + k + 1;
            const double vj = vs[j], wj = ws[j];
            for (int i = lane; i < m; i += 32) col[i] -= vs[i] * wj + ws[i] * vj;
        }
        gsync();
    }
    if (GRID ? blockIdx.x == 0 && tid == 0 : tid == 0) {
        if (n >= 2) {
            dout[n - 2] = A[(size_t)(n - 2) * n + n - 2];
            eout[n - 2] = A[(size_t)(n - 2) * n + n - 1];
        }
        dout[n - 1] = A[(size_t)(n - 1) * n + n - 1];
    }
}

// Eigenvalue j (ascending) of the tridiagonal (d, e) by 33-section: each lane of the warp evaluates
// the Sturm count (number of eigenvalues < x) at one interior point of the current bracket, which
// shrinks 33x per round.  The count uses the LDL^T pivot recurrence q_i = d_i - x - e_{i-1}^2 / q_{i-1}
// with tiny pivots replaced by -pivmin (the standard guard).  Deterministic; accuracy ~ eps ||T||.
__global__ void __launch_bounds__(256) k_tri_multisect(int n, const double* __restrict__ d,
                                                        const double* __restrict__ e, double* __restrict__ w) {
    extern __shared__ double tm[];
    double* ds = tm;
    double* e2 = tm + n;
    const int tid = threadIdx.x, lane = tid & 31;
    for (int i = tid; i < n; i += blockDim.x) {
        ds[i] = d[i];
        e2[i] = i + 1 < n ? e[i] * e[i] : 0.0;
    }
    __syncthreads();
    // Gershgorin bracket and pivot guard (identical in every warp)
    double lo = 1e300, hi = -1e300, emax = 0.0;
    for (int i = 0; i < n; ++i) {
        const double r = (i > 0 ? sqrt(e2[i - 1]) : 0.0) + (i + 1 < n ? sqrt(e2[i]) : 0.0);
        lo = fmin(lo, ds[i] - r);
        hi = fmax(hi, ds[i] + r);
        emax = fmax(emax, e2[i]);
    }
    const double nrm = fmax(fabs(lo), fabs(hi));
    const double pivmin = 2.2250738585072014e-308 * fmax(1.0, emax) * 1e10;
    lo -= 4.0 * 2.220446049250313e-16 * nrm + pivmin;
    hi += 4.0 * 2.220446049250313e-16 * nrm + pivmin;
    const int j = blockIdx.x * (blockDim.x >> 5) + (tid >> 5);
    if (j >= n) return;
    if (nrm == 0.0) {  // T = 0: every eigenvalue is exactly zero
        if (lane == 0) w[j] = 0.0;
        return;
    }
    for (int it = 0; it < 14; ++it) {
        const double x = lo + (hi - lo) * (double)(lane + 1) * (1.0 / 33.0);
        int cnt = 0;
        double q = ds[0] - x;
        if (fabs(q) < pivmin) q = -pivmin;
        cnt += q < 0.0;
        for (int i = 1; i < n; ++i) {
            q = ds[i] - x - e2[i - 1] / q;
            if (fabs(q) < pivmin) q = -pivmin;
            cnt += q < 0.0;
        }
        // bracket: last point with count <= j (new lo), first point with count > j (new hi)
        const unsigned above = __ballot_sync(0xffffffffu, cnt > j);
        const int first = above ? __ffs(above) - 1 : 32;
        const double xlo = __shfl_sync(0xffffffffu, x, first > 0 ? first - 1 : 0);
        const double xhi = __shfl_sync(0xffffffffu, x, first < 32 ? first : 31);
        if (first > 0) lo = xlo;
        if (first < 32) hi = xhi;
        if (hi - lo <= 2.220446049250313e-16 * fmax(fabs(lo), fabs(hi))) break;
    }
    if (lane == 0) w[j] = 0.5 * (lo + hi);
}

static void sym_eigvals_tridiag(acp_context* ctx, double* A, int n, double* w) {
    double* d = ctx->wsd("eig_d", n);
    double* e = ctx->wsd("eig_e", n);
    double* p = ctx->wsd("eig_p", n);
    const size_t small = ((size_t)2 * n + 32 + (size_t)n * n) * sizeof(double);
    if (small <= 200 * 1024) {
        func_attr((const void*)k_tridiag<false>, 200 * 1024);
        const int nt = std::min(1024, std::max(128, cdiv(n, 32) * 32 * 4));
        k_tridiag<false><<<1, nt, small, ctx->stream>>>(A, n, p, d, e);
    } else {
        const size_t smem = ((size_t)2 * n + 32) * sizeof(double);
        const void* fn = (const void*)k_tridiag<true>;
        if (smem > 48 * 1024) func_attr(fn, smem);
        int occ = 0;
        ACP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
        int dev = 0, sms = 0;
        ACP_CUDA(cudaGetDevice(&dev));
        ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        ACP_REQUIRE(occ >= 1, "tridiag: cooperative kernel does not fit");
        // one warp per trailing column at the first step, at most one CTA per SM
        const int G = std::max(1, std::min(sms, cdiv(n, 8)));
        void* args[] = {&A, &n, &p, &d, &e};
        ACP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(256), args, smem, ctx->stream));
    }
    launched(ctx);
    const size_t ms = (size_t)2 * n * sizeof(double);
    ACP_REQUIRE(ms <= 200 * 1024, "eigenvalue search: n too large");
    if (ms > 48 * 1024) {
        func_attr((const void*)k_tri_multisect, 200 * 1024);
    }
    k_tri_multisect<<<cdiv(n, 8), 256, ms, ctx->stream>>>(n, d, e, w);
    launched(ctx);
}

void sym_eig(acp_context* ctx, double* A, int n, double* w, double* V) {
    // eigenvalues only: tridiagonalisation + multisection (ACP_EIG_JACOBI=1 selects the one-warp
    // Jacobi for n <= 32, ACP_EIG_BLOCK=1 the block Jacobi -- kept as tested alternatives)
    if (!V && n <= 32 && getenv("ACP_EIG_JACOBI")) {
        k_jacobi_warp<<<1, 32, 0, ctx->stream>>>(A, n, w, 40);
        launched(ctx);
        return;
    }
    if (!V && !getenv("ACP_EIG_BLOCK")) {
        sym_eigvals_tridiag(ctx, A, n, w);
        return;
    }
    double* Vt = V ? ctx->wsd("eig_Vt", (size_t)n * n) : nullptr;
    int* order = ctx->wsi("eig_order", n + 2);
    double* rot = ctx->wsd("eig_rot", 4 * (size_t)(n / 2 + 2));
    const size_t bytes = (size_t)n * n * sizeof(double);
    const int use_smem = bytes <= 200 * 1024;
    func_attr((const void*)k_jacobi, 200 * 1024);
    // one warp per rotation pair (n/2 pairs) is enough; fewer threads make each barrier cheaper
    const int jt = std::min(1024, std::max(64, ((n + 1) / 2) * 32));
    k_jacobi<<<1, jt, use_smem ? bytes : 0, ctx->stream>>>(A, n, Vt, w, order, rot, 40, use_smem);
    launched(ctx);
    if (V) {
        k_permute_cols<<<cdiv((long long)n * n, 256), 256, 0, ctx->stream>>>(n, Vt, order, V);
        launched(ctx);
    }
}

// Right-looking Cholesky, lower triangle; status 1 if not positive definite.
__global__ void __launch_bounds__(1024) k_cholesky(double* __restrict__ A, int n, int* __restrict__ status) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int k = 0; k < n; ++k) {
        const double d = A[(size_t)k * n + k];
        if (d <= 0.0) {
            if (tid == 0) *status = 1;
            return;
        }
        const double r = sqrt(d);
        __syncthreads();
        if (tid == 0) A[(size_t)k * n + k] = r;
        for (int i = k + 1 + tid; i < n; i += nt) A[(size_t)k * n + i] /= r;
        __syncthreads();
        const int rows = n - k - 1;
        const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
        for (int jj = warp; jj < rows; jj += nwarp) {
            const int j = k + 1 + jj;
            const double ljk = A[(size_t)k * n + j];
            for (int i = j + lane; i < n; i += 32) A[(size_t)j * n + i] -= A[(size_t)k * n + i] * ljk;
        }
        __syncthreads();
    }
    for (long long e = tid; e < (long long)n * n; e += nt) {
        const int i = (int)(e % n), j = (int)(e / n);
        if (j > i) A[e] = 0.0;
    }
    if (tid == 0) *status = 0;
}

void cholesky(acp_context* ctx, double* A, int n) {
    int* st = ctx->wsi("chol_status", 1);
    k_cholesky<<<1, 1024, 0, ctx->stream>>>(A, n, st);
    launched(ctx);
    int h = 0;
    ACP_CUDA(cudaMemcpyAsync(&h, st, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h != 0) throw Error(ACP_ERR_SINGULAR, "Cholesky: matrix not positive definite");
}

}  // namespace acp
