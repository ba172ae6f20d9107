// qrcp.cu -- Alg. 2 with Remark 1 on the GPU.
//
//  K4  G~ = G' Omega            real SRFT of the perturbation columns (DMMA GEMM)
//  K5  M~^T(i + q N_occ, a) = psi_i(a) G~(a, q)   Kronecker rows
//  K6  pivoted QR of M~^T: greedy max-norm pivot among the remaining columns
//      (lowest position on ties), Householder reflection, trailing update with exact
//      norm recomputation -- ONE persistent cooperative kernel, columns resident in
//      shared memory, one grid barrier per pivot (see k_qrcp_persistent)
//  K7  Xi^T = R11^{-1} R_{1:N,:} Pi^{-1}: warp-per-column back
//      substitution + scatter.
#include <cooperative_groups.h>

#include "gemm.cuh"

#include <algorithm>
#include <cmath>
#include <vector>
#include <cstdlib>
#include <cstdio>

namespace acp {

// Omega(I, 2q) + i Omega(I, 2q+1) = exp(-2 pi i I nu_q / n) exp(2 pi i theta_I),  I = 1..n.
__global__ void k_srft_omega(int n, int r_half, const double* __restrict__ theta, const int* __restrict__ nu,
                             double* __restrict__ Om) {
    int I0 = blockIdx.x * blockDim.x + threadIdx.x;  // 0-based row
    int q = blockIdx.y;
    if (I0 >= n || q >= r_half) return;
    long long Inu = (long long)(I0 + 1) * (long long)nu[q];
    Inu %= n;
    double frac = theta[I0] - (double)Inu / (double)n;  // turns
    double s, c;
    sincospi(2.0 * frac, &s, &c);
    Om[(size_t)(2 * q) * n + I0] = c;
    Om[(size_t)(2 * q + 1) * n + I0] = s;
}

// A (m x Ng, ld m), m = n_occ * r:  A[i + q n_occ, a] = Psi(a, i) Gt(a, q).  32 grid points per CTA.
__global__ void __launch_bounds__(256) k_kron_rows(int Ng, int n_occ, int r, const double* __restrict__ Psi,
                                                   const double* __restrict__ Gt, double* __restrict__ A) {
    extern __shared__ double sm[];
    double* sp = sm;                 // 32 x n_occ  (a-major)
    double* sg = sm + 32 * n_occ;    // 32 x r
    const int a0 = blockIdx.x * 32;
    for (int idx = threadIdx.x; idx < 32 * n_occ; idx += blockDim.x) {
        int aa = idx % 32, i = idx / 32;
        sp[aa * n_occ + i] = (a0 + aa < Ng) ? Psi[(size_t)i * Ng + a0 + aa] : 0.0;
    }
    for (int idx = threadIdx.x; idx < 32 * r; idx += blockDim.x) {
        int aa = idx % 32, q = idx / 32;
        sg[aa * r + q] = (a0 + aa < Ng) ? Gt[(size_t)q * Ng + a0 + aa] : 0.0;
    }
    __syncthreads();
    const int m = n_occ * r;
    for (int aa = 0; aa < 32 && a0 + aa < Ng; ++aa) {
        double* col = A + (size_t)(a0 + aa) * m;
        for (int idx = threadIdx.x; idx < m; idx += blockDim.x) {
            int i = idx % n_occ, q = idx / n_occ;
            col[idx] = sp[aa * n_occ + i] * sg[aa * r + q];
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent pivoted QR: ONE cooperative launch for the whole factorisation.
// CTA b owns the grid-point columns [b*cpb, (b+1)*cpb) for the entire run (in shared memory
// when they fit, else in place in global memory/L2); columns never move -- a position map
// reproduces the swap semantics of column-pivoted QR (ties -> lowest current position).
// Per step j there is exactly one grid barrier:
//   every CTA publishes its best candidate (norm^2, position, column) and a copy of that
//   column's rows j..m-1 (double-buffered by step parity), grid.sync(), then every CTA
//   redundantly selects the same winner, builds the same Householder vector from the
//   published copy, and updates its own remaining columns (exact norm recomputation).
struct QrSlot {
    double n2;
    int pos;
    int col;
};

// Warp index that the compiler can prove warp-uniform (a shuffle from lane 0): branches and
// loops on it stay convergent, so the __shfl_sync calls inside them compile to plain SHFL
// instead of the WARPSYNC.COLLECTIVE emulation used for possibly-divergent code.
__device__ __forceinline__ int uniform_warp() { return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0); }

// Householder update of a CTA's owned, not-yet-pivoted columns, two columns per warp (16 lanes
// each; warp-uniform loop, predicated work, full-warp shuffles).  Column `cw` (global index) is
// the pivot: it becomes (alpha, 0, ...).  v (rows j..m-1) and tau are shared by the CTA; n2[lc]
// receives the exact trailing norm^2 (rows j+1..m-1).  Summation order is fixed.
template <class ColP>
__device__ __forceinline__ void qr_update_cols(ColP colp, int warp, int nc, int c0, int cw, int j, int m,
                                               double alpha, double tau, const double* __restrict__ v,
                                               const int* __restrict__ dn, double* __restrict__ n2) {
    const int nwarp = blockDim.x >> 5;
    const int h = (threadIdx.x >> 4) & 1, q = threadIdx.x & 15;
    for (int base = 2 * warp; base < nc; base += 2 * nwarp) {
        const int lc = base + h;
        const bool valid = lc < nc;
        const bool piv = valid && (c0 + lc == cw);
        const bool live = valid && !piv && !dn[lc];
        double* c = colp(valid ? lc : base);
        double d = 0.0;
        if (live)
            for (int i = j + q; i < m; i += 16) d += v[i] * c[i];
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        const double f = tau * d;
        double nn = 0.0;
        if (live) {
            for (int i = j + q; i < m; i += 16) {
                const double y = c[i] - f * v[i];
                c[i] = y;
                if (i > j) nn += y * y;
            }
        } else if (piv) {
            for (int i = j + q; i < m; i += 16) c[i] = (i == j) ? alpha : 0.0;
        }
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
        if (live && q == 0) n2[lc] = nn;
    }
}

// Global-memory variant for long columns (m <= 32*KR): ONE warp per column with the column's
// trailing rows in registers (lane l: rows l, l+32, ...), so a step reads and writes each column
// once with KR independent loads in flight per lane -- the 16-lane version above re-reads the
// column for the update and keeps too few loads in flight to reach HBM bandwidth.
template <int KR, class ColP>
__device__ __forceinline__ void qr_update_cols_warp(ColP colp, int warp, int nc, int c0, int cw, int j, int m,
                                                    double alpha, double tau, const double* __restrict__ v,
                                                    const int* __restrict__ dn, double* __restrict__ n2) {
    // two columns per warp and iteration (lc, lc + nwarp): two independent load batches in flight
    const int nwarp = blockDim.x >> 5, lane = threadIdx.x & 31;
    for (int lc0 = warp; lc0 < nc; lc0 += 2 * nwarp) {
        const int lc1 = lc0 + nwarp;
        const bool has1 = lc1 < nc;
        const bool piv0 = c0 + lc0 == cw, piv1 = has1 && c0 + lc1 == cw;
        const bool live0 = !piv0 && !dn[lc0];
        const bool live1 = has1 && !piv1 && !dn[lc1];
        double* ca = colp(lc0);
        double* cb = colp(has1 ? lc1 : lc0);
        double ya[KR], yb[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int i = lane + 32 * k;
            const bool in = i >= j && i < m;
            ya[k] = (live0 && in) ? ca[i] : 0.0;
            yb[k] = (live1 && in) ? cb[i] : 0.0;
        }
        double da = 0.0, db = 0.0;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int i = lane + 32 * k;
            if (i >= j && i < m) {
                const double vi = v[i];
                da += vi * ya[k];
                db += vi * yb[k];
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            da += __shfl_xor_sync(0xffffffffu, da, o);
            db += __shfl_xor_sync(0xffffffffu, db, o);
        }
        const double fa = tau * da, fb = tau * db;
        double na = 0.0, nb = 0.0;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int i = lane + 32 * k;
            if (i >= j && i < m) {
                const double vi = v[i];
                const double ua = ya[k] - fa * vi, ub = yb[k] - fb * vi;
                if (live0) ca[i] = ua;
                if (live1) cb[i] = ub;
                if (i > j) {
                    na += ua * ua;
                    nb += ub * ub;
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            na += __shfl_xor_sync(0xffffffffu, na, o);
            nb += __shfl_xor_sync(0xffffffffu, nb, o);
        }
        if (lane == 0) {
            if (live0) n2[lc0] = na;
            if (live1) n2[lc1] = nb;
        }
        if (piv0)
            for (int i = j + lane; i < m; i += 32) ca[i] = (i == j) ? alpha : 0.0;
        if (piv1)
            for (int i = j + lane; i < m; i += 32) cb[i] = (i == j) ? alpha : 0.0;
    }
}

template <int KR, class ColP>
__device__ __forceinline__ void qr_update_cols_warp1(ColP colp, int warp, int nc, int c0, int cw, int j, int m,
                                                     double alpha, double tau, const double* __restrict__ v,
                                                     const int* __restrict__ dn, double* __restrict__ n2) {
    const int nwarp = blockDim.x >> 5, lane = threadIdx.x & 31;
    for (int lc = warp; lc < nc; lc += nwarp) {
        const bool piv = c0 + lc == cw;
        const bool live = !piv && !dn[lc];
        double* c = colp(lc);
        if (live) {
            double y[KR];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = lane + 32 * k;
                y[k] = (i >= j && i < m) ? c[i] : 0.0;
            }
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = lane + 32 * k;
                if (i >= j && i < m) d += v[i] * y[k];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const double f = tau * d;
            double nn = 0.0;
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = lane + 32 * k;
                if (i >= j && i < m) {
                    const double yy = y[k] - f * v[i];
                    c[i] = yy;
                    if (i > j) nn += yy * yy;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
            if (lane == 0) n2[lc] = nn;
        } else if (piv) {
            for (int i = j + lane; i < m; i += 32) c[i] = (i == j) ? alpha : 0.0;
        }
    }
}

// Long columns (m > 2048, configs[4]: m = 4096): one warp per column in chunks of 32 KR rows --
// pass 1 accumulates v.c chunk by chunk (KR loads in flight per lane), pass 2 re-reads each chunk,
// updates, stores and accumulates the new norm.  Two reads + one write per element, like the
// 16-lane version, but with enough loads in flight to run at HBM bandwidth.
template <int KR, class ColP>
__device__ __forceinline__ void qr_update_cols_chunked(ColP colp, int warp, int nc, int c0, int cw, int j, int m,
                                                       double alpha, double tau, const double* __restrict__ v,
                                                       const int* __restrict__ dn, double* __restrict__ n2) {
    const int nwarp = blockDim.x >> 5, lane = threadIdx.x & 31;
    const int r_begin = j & ~31;
    for (int lc = warp; lc < nc; lc += nwarp) {
        const bool piv = c0 + lc == cw;
        const bool live = !piv && !dn[lc];
        double* c = colp(lc);
        if (live) {
            double d = 0.0;
            for (int r0 = r_begin; r0 < m; r0 += 32 * KR) {
                double y[KR];
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const int i = r0 + lane + 32 * k;
                    y[k] = (i >= j && i < m) ? c[i] : 0.0;
                }
                asm volatile("" ::: "memory");  // issue all KR loads before their first use
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const int i = r0 + lane + 32 * k;
                    if (i >= j && i < m) d += v[i] * y[k];
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const double f = tau * d;
            double nn = 0.0;
            for (int r0 = r_begin; r0 < m; r0 += 32 * KR) {
                double y[KR];
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const int i = r0 + lane + 32 * k;
                    y[k] = (i >= j && i < m) ? c[i] : 0.0;
                }
                asm volatile("" ::: "memory");  // issue all KR loads before their first use
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const int i = r0 + lane + 32 * k;
                    if (i >= j && i < m) {
                        const double yy = y[k] - f * v[i];
                        c[i] = yy;
                        if (i > j) nn += yy * yy;
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
            if (lane == 0) n2[lc] = nn;
        } else if (piv) {
            for (int i = j + lane; i < m; i += 32) c[i] = (i == j) ? alpha : 0.0;
        }
    }
}

// Two columns per warp variant of the chunked update (independent load streams interleave).
template <int KR, class ColP>
__device__ __forceinline__ void qr_update_cols_chunked2(ColP colp, int warp, int nc, int c0, int cw, int j, int m,
                                                        double alpha, double tau, const double* __restrict__ v,
                                                        const int* __restrict__ dn, double* __restrict__ n2) {
    const int nwarp = blockDim.x >> 5, lane = threadIdx.x & 31;
    const int r_begin = j & ~31;
    for (int lc0 = warp; lc0 < nc; lc0 += 2 * nwarp) {
        const int lc1 = lc0 + nwarp;
        const bool has1 = lc1 < nc;
        const bool piv0 = c0 + lc0 == cw, piv1 = has1 && c0 + lc1 == cw;
        const bool live0 = !piv0 && !dn[lc0];
        const bool live1 = has1 && !piv1 && !dn[lc1];
        double* ca = colp(lc0);
        double* cb = colp(has1 ? lc1 : lc0);
        double da = 0.0, db = 0.0;
        for (int r0 = r_begin; r0 < m; r0 += 32 * KR) {
            double ya[KR], yb[KR];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = r0 + lane + 32 * k;
                const bool in = i >= j && i < m;
                ya[k] = (live0 && in) ? ca[i] : 0.0;
                yb[k] = (live1 && in) ? cb[i] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = r0 + lane + 32 * k;
                if (i >= j && i < m) {
                    const double vi = v[i];
                    da += vi * ya[k];
                    db += vi * yb[k];
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            da += __shfl_xor_sync(0xffffffffu, da, o);
            db += __shfl_xor_sync(0xffffffffu, db, o);
        }
        const double fa = tau * da, fb = tau * db;
        double na = 0.0, nb = 0.0;
        for (int r0 = r_begin; r0 < m; r0 += 32 * KR) {
            double ya[KR], yb[KR];
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = r0 + lane + 32 * k;
                const bool in = i >= j && i < m;
                ya[k] = (live0 && in) ? ca[i] : 0.0;
                yb[k] = (live1 && in) ? cb[i] : 0.0;
            }
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int i = r0 + lane + 32 * k;
                if (i >= j && i < m) {
                    const double vi = v[i];
                    const double ua = ya[k] - fa * vi, ub = yb[k] - fb * vi;
                    if (live0) ca[i] = ua;
                    if (live1) cb[i] = ub;
                    if (i > j) {
                        na += ua * ua;
                        nb += ub * ub;
                    }
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            na += __shfl_xor_sync(0xffffffffu, na, o);
            nb += __shfl_xor_sync(0xffffffffu, nb, o);
        }
        if (lane == 0) {
            if (live0) n2[lc0] = na;
            if (live1) n2[lc1] = nb;
        }
        if (piv0)
            for (int i = j + lane; i < m; i += 32) ca[i] = (i == j) ? alpha : 0.0;
        if (piv1)
            for (int i = j + lane; i < m; i += 32) cb[i] = (i == j) ? alpha : 0.0;
    }
}

template <bool SMEM, int KR>
__global__ void __launch_bounds__(256) k_qrcp_persistent(int m, int Ng, double* __restrict__ Ag, int kmax, double eps,
                                                         int fixed, QrSlot* __restrict__ slots,
                                                         double* __restrict__ cand, int* __restrict__ perm,
                                                         double* __restrict__ rdiag, int* __restrict__ out_nmu) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double qsm[];
    __shared__ double red_d[32];
    __shared__ int red_i[32];
    __shared__ int red_j[32];
    __shared__ int s_lc;
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = uniform_warp(), nwarp = blockDim.x >> 5;
    const int cpb = (Ng + G - 1) / G;
    const int c0 = b * cpb;
    const int nc = max(0, min(Ng, c0 + cpb) - c0);
    double* cols = qsm;
    double* v = qsm + (SMEM ? (size_t)cpb * m : 0);
    double* n2 = v + m;
    int* pos = reinterpret_cast<int*>(n2 + cpb);
    int* dn = pos + cpb;
    auto colp = [&](int lc) -> double* { return SMEM ? cols + (size_t)lc * m : Ag + (size_t)(c0 + lc) * m; };
    if (SMEM)
        for (int e = tid; e < nc * m; e += blockDim.x) cols[e] = Ag[(size_t)c0 * m + e];
    __syncthreads();
    for (int lc = warp; lc < nc; lc += nwarp) {
        const double* c = colp(lc);
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += c[i] * c[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            n2[lc] = s;
            pos[lc] = c0 + lc;
            dn[lc] = 0;
        }
    }
    __syncthreads();
    double r11 = 0.0;
    int N = kmax;
    for (int j = 0; j < kmax; ++j) {
        const int buf = j & 1;
        // ---- local candidate: max n2, ties -> lowest position
        if (warp == 0) {
            double bn = -1.0;
            int bp = 1 << 30, bl = -1;
            for (int lc = lane; lc < nc; lc += 32) {
                if (dn[lc]) continue;
                const double x = n2[lc];
                if (x > bn || (x == bn && pos[lc] < bp)) {
                    bn = x;
                    bp = pos[lc];
                    bl = lc;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bl = ol;
                }
            }
            if (lane == 0) {
                s_lc = bl;
                QrSlot sl;
                sl.n2 = bn;
                sl.pos = bp;
                sl.col = bl >= 0 ? c0 + bl : -1;
                slots[buf * G + b] = sl;
            }
        }
        __syncthreads();
        if (s_lc >= 0) {
            const double* c = colp(s_lc);
            double* dst = cand + ((size_t)buf * G + b) * m;
            for (int i = j + tid; i < m; i += blockDim.x) dst[i] = c[i];
        }
        __threadfence();
        grid.sync();
        __syncthreads();  // re-establishes (for the compiler) a convergent block after grid.sync
        // ---- global winner (identical in every CTA)
        double bn = -1.0;
        int bp = 1 << 30, bs = -1;
        for (int s = tid; s < G; s += blockDim.x) {
            // L2 reads (ld.cg): the slots were written by other CTAs; L1 is not coherent
            const double sn = __ldcg(&slots[buf * G + s].n2);
            const int sp = __ldcg(&slots[buf * G + s].pos);
            const int sc = __ldcg(&slots[buf * G + s].col);
            if (sc >= 0 && (sn > bn || (sn == bn && sp < bp))) {
                bn = sn;
                bp = sp;
                bs = s;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double on = __shfl_xor_sync(0xffffffffu, bn, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            const int os = __shfl_xor_sync(0xffffffffu, bs, o);
            if (on > bn || (on == bn && op < bp)) {
                bn = on;
                bp = op;
                bs = os;
            }
        }
        if (lane == 0) {
            red_d[warp] = bn;
            red_i[warp] = bp;
            red_j[warp] = bs;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 1; w < nwarp; ++w)
                if (red_d[w] > red_d[0] || (red_d[w] == red_d[0] && red_i[w] < red_i[0])) {
                    red_d[0] = red_d[w];
                    red_i[0] = red_i[w];
                    red_j[0] = red_j[w];
                }
        }
        __syncthreads();
        const double wn2 = red_d[0];
        const int pw = red_i[0], ws = red_j[0];
        const double rjj = sqrt(fmax(wn2, 0.0));
        if (j == 0) r11 = rjj;
        // block-uniform exit (__syncthreads_or), so the code after the loop stays convergent
        if (__syncthreads_or(ws < 0 || rjj == 0.0 || (fixed <= 0 && rjj < eps * r11))) {
            N = j;
            break;
        }
        const int cw = __ldcg(&slots[buf * G + ws].col);
        // ---- Householder vector from the published copy of the winner column
        const double* x = cand + ((size_t)buf * G + ws) * m;
        double s = 0.0;
        for (int i = j + tid; i < m; i += blockDim.x) {
            const double xi = __ldcg(x + i);
            v[i] = xi;
            s += xi * xi;
        }
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        __syncthreads();
        if (lane == 0) red_d[warp] = s;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < nwarp; ++w) t += red_d[w];
            red_d[0] = t;
        }
        __syncthreads();
        const double xn2 = red_d[0];
        const double xn = sqrt(xn2);
        const double x0 = v[j];
        const double alpha = (x0 >= 0.0) ? -xn : xn;
        const double v0 = x0 - alpha;
        const double tau = 2.0 / (xn2 - x0 * x0 + v0 * v0);
        __syncthreads();
        if (tid == 0) v[j] = v0;
        if (b == 0 && tid == 0) rdiag[j] = xn;
        // ---- position bookkeeping (swap of positions j and pw) and the pivot column itself
        for (int lc = tid; lc < nc; lc += blockDim.x) {
            if (c0 + lc == cw) {
                pos[lc] = j;
                dn[lc] = 1;
            } else if (!dn[lc] && pos[lc] == j) {
                pos[lc] = pw;
            }
        }
        __syncthreads();
        // ---- trailing update of the remaining owned columns (16 threads per column)
        if constexpr (KR == 32)  // two columns per warp (243 registers)
            qr_update_cols_warp<32>(colp, warp, nc, c0, cw, j, m, alpha, tau, v, dn, n2);
        else if constexpr (KR == 64)
            qr_update_cols_warp1<64>(colp, warp, nc, c0, cw, j, m, alpha, tau, v, dn, n2);
        else if constexpr (KR == 1)  // m > 2048: warp per column, 1024-row chunks
            qr_update_cols_chunked<32>(colp, warp, nc, c0, cw, j, m, alpha, tau, v, dn, n2);
        else if constexpr (KR == 2)  // m > 2048: two columns per warp, 512-row chunks
            qr_update_cols_chunked2<16>(colp, warp, nc, c0, cw, j, m, alpha, tau, v, dn, n2);
        else
            qr_update_cols(colp, warp, nc, c0, cw, j, m, alpha, tau, v, dn, n2);
        __syncthreads();
    }
    if (SMEM)
        for (int e = tid; e < nc * m; e += blockDim.x) Ag[(size_t)c0 * m + e] = cols[e];
    for (int lc = tid; lc < nc; lc += blockDim.x) perm[pos[lc]] = c0 + lc;
    if (b == 0 && tid == 0) *out_nmu = N;
}

// ---------------------------------------------------------------------------
// Cluster QRCP for problems that fit in the shared memory of one thread-block cluster
// (N_g * m * 8 B <= ~16 x 190 KB; configs[0..1] and small 2D): the same algorithm and tie
// rules as k_qrcp_persistent, with the per-pivot exchange through distributed shared memory
// and ONE cluster barrier per pivot:
//   * each CTA finds its local best column (warp 0), PUSHES its (norm^2, position, column)
//     slot into every peer's slot table (DSMEM stores) and copies the candidate's rows j..m-1
//     into a parity-double-buffered publish buffer of its own shared memory;
//   * cluster barrier; every CTA selects the same winner from its LOCAL slot table, then reads
//     the winner's published copy through DSMEM (the only remote read of the step);
//   * |R_jj| is the winner's exact trailing norm (recomputed in the previous step), and the
//     Householder update of the owned columns is one pass per column with the column's rows in
//     registers (16 lanes per column): dot, shuffle reduction, update + new exact norm.
// A slot / publish buffer of parity j is rewritten only at step j+2, after another barrier.
template <int MAXK>
__global__ void __launch_bounds__(1024) k_qrcp_cluster(int m, int Ng, double* __restrict__ Ag, int kmax, double eps,
                                                      int fixed, int* __restrict__ perm, double* __restrict__ rdiag,
                                                      int* __restrict__ out_nmu, long long* __restrict__ tprof) {
    // tprof (debug, may be null): per step j, clock64() at phase boundaries of CTA 0 / thread 0
#define QR_TP(k) \
    if (tprof && blockIdx.x == 0 && threadIdx.x == 0 && j < 512) tprof[8 * j + (k)] = clock64();
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double csm[];
    __shared__ QrSlot allslot[2][16];  // [parity][source rank], filled by the peers' pushes
    __shared__ double s_wn2;
    __shared__ int s_pos, s_rank, s_col, s_lc;
    const int CS = (int)cl.num_blocks(), b = (int)cl.block_rank(), tid = threadIdx.x;
    const int lane = tid & 31, warp = uniform_warp(), nwarp = blockDim.x >> 5;
    const int cpb = (Ng + CS - 1) / CS;
    const int c0 = b * cpb;
    const int nc = max(0, min(Ng, c0 + cpb) - c0);
    double* cols = csm;                         // cpb x m
    double* v = cols + (size_t)cpb * m;         // m
    double* pub = v + m;                        // 2 x m published candidate copies
    double* n2 = pub + 2 * (size_t)m;           // cpb
    int* pos = reinterpret_cast<int*>(n2 + cpb);
    int* dn = pos + cpb;
    for (int e = tid; e < nc * m; e += blockDim.x) cols[e] = Ag[(size_t)c0 * m + e];
    __syncthreads();
    for (int lc = warp; lc < nc; lc += nwarp) {
        const double* c = cols + (size_t)lc * m;
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s += c[i] * c[i];
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            n2[lc] = s;
            pos[lc] = c0 + lc;
            dn[lc] = 0;
        }
    }
    __syncthreads();
    double r11 = 0.0;
    int N = kmax;
    cl.sync();  // every CTA of the cluster has started before the first DSMEM push
    for (int j = 0; j < kmax; ++j) {
        const int buf = j & 1;
        QR_TP(0)
        if (warp == 0) {
            double bn = -1.0;
            int bp = 1 << 30, bl = -1;
            for (int lc = lane; lc < nc; lc += 32) {
                if (dn[lc]) continue;
                const double x = n2[lc];
                if (x > bn || (x == bn && pos[lc] < bp)) {
                    bn = x;
                    bp = pos[lc];
                    bl = lc;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {  // butterfly: every lane ends with the result
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bl = ol;
                }
            }
            QrSlot sl;
            sl.n2 = bn;
            sl.pos = bp;
            sl.col = bl >= 0 ? c0 + bl : -1;
            if (lane < CS) cl.map_shared_rank(&allslot[0][0], lane)[buf * 16 + b] = sl;  // push to peer `lane`
            if (lane == 0) s_lc = bl;
        }
        __syncthreads();
        if (s_lc >= 0) {
            const double* c = cols + (size_t)s_lc * m;
            for (int i = j + tid; i < m; i += blockDim.x) pub[(size_t)buf * m + i] = c[i];
        }
        cl.sync();
        QR_TP(1)
        if (warp == 0) {
            double bn = -1.0;
            int bp = 1 << 30, bs = -1, bc = -1;
            if (lane < CS) {
                const QrSlot sl = allslot[buf][lane];
                if (sl.col >= 0) {
                    bn = sl.n2;
                    bp = sl.pos;
                    bs = lane;
                    bc = sl.col;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int os = __shfl_xor_sync(0xffffffffu, bs, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bs = os;
                    bc = oc;
                }
            }
            if (lane == 0) {
                s_wn2 = bn;
                s_pos = bp;
                s_rank = bs;
                s_col = bc;
            }
        }
        __syncthreads();
        const double wn2 = s_wn2;
        const int pw = s_pos, ws = s_rank, cw = s_col;
        const double rjj = sqrt(fmax(wn2, 0.0));
        if (j == 0) r11 = rjj;
        // block-uniform exit (__syncthreads_or), so the code after the loop stays convergent
        if (__syncthreads_or(ws < 0 || rjj == 0.0 || (fixed <= 0 && rjj < eps * r11))) {
            N = j;
            break;
        }
        QR_TP(2)
        // ---- Householder vector: the winner's published rows j..m-1 (one DSMEM read); row j of
        // v holds v0 = x0 - alpha directly, so the update below has no per-element selects
        const double* x = cl.map_shared_rank(pub, ws) + (size_t)buf * m;
        const double x0 = x[j];
        const double alpha = (x0 >= 0.0) ? -rjj : rjj;
        const double v0 = x0 - alpha;
        const double tau = 2.0 / (wn2 - x0 * x0 + v0 * v0);
        for (int i = j + tid; i < m; i += blockDim.x) v[i] = (i == j) ? v0 : x[i];
        if (b == 0 && tid == 0) rdiag[j] = rjj;
        __syncthreads();
        QR_TP(3)
        // ---- fused single-pass update: one column per warp, rows i = j + lane + 32k in registers
        const int kc = (m - j - lane + 31) >> 5;  // rows of this lane (<= MAXK)
        for (int lc = warp; lc < nc; lc += nwarp) {
            double* c = cols + (size_t)lc * m + j + lane;
            const double* vv = v + j + lane;
            if (c0 + lc == cw) {
#pragma unroll
                for (int k = 0; k < MAXK; ++k)
                    if (k < kc) c[32 * k] = (k == 0 && lane == 0) ? alpha : 0.0;
                if (lane == 0) {
                    pos[lc] = j;
                    dn[lc] = 1;
                }
                continue;  // warp-uniform
            }
            if (dn[lc]) continue;  // warp-uniform
            double y[MAXK];
            double d = 0.0;
#pragma unroll
            for (int k = 0; k < MAXK; ++k) {
                y[k] = k < kc ? c[32 * k] : 0.0;
                d += (k < kc ? vv[32 * k] : 0.0) * y[k];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
            const double f = tau * d;
            double nn = 0.0;
#pragma unroll
            for (int k = 0; k < MAXK; ++k) {
                if (k < kc) {
                    const double yy = y[k] - f * vv[32 * k];
                    c[32 * k] = yy;
                    if (k > 0 || lane > 0) nn += yy * yy;  // trailing rows j+1..m-1 only
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
            if (lane == 0) {
                n2[lc] = nn;
                if (pos[lc] == j) pos[lc] = pw;  // swap semantics of column pivoting
            }
        }
        __syncthreads();
        QR_TP(4)
    }
    for (int e = tid; e < nc * m; e += blockDim.x) Ag[(size_t)c0 * m + e] = cols[e];
    for (int lc = tid; lc < nc; lc += blockDim.x) perm[pos[lc]] = c0 + lc;
    if (b == 0 && tid == 0) *out_nmu = N;
    cl.sync();  // peers may still be reading this CTA's buffers when it leaves the loop
}

// ---------------------------------------------------------------------------
// Cluster QRCP with REGISTER-RESIDENT columns (problems with N_g/CS <= 16*CPW columns per CTA
// and m <= 32*KR rows): the same algorithm, exchange and tie rules as k_qrcp_cluster, but each
// CTA's columns never leave registers -- warp w owns local columns w, w+16, ..., lane l rows
// l, l+32, ... -- so a pivot step moves no column data through shared memory: each lane reads
// its KR entries of the Householder vector once per step and updates CPW columns in registers
// (v is zero above row j, so rows < j are untouched without any masking).  512 threads.
// Reduce-scatter of 8 per-lane values over a warp in 9 shuffles (instead of 8 x 5): halving
// exchanges over lane bits 0..2, then a plain butterfly over bits 3..4.  Afterwards lane l holds
// the warp total of value index rs8_index(l); every copy of a total is bitwise identical (each
// level adds the same two partial sums, in commutative order).
__device__ __forceinline__ int rs8_index(int l) { return ((l & 1) << 2) | (l & 2) | ((l >> 2) & 1); }
__device__ __forceinline__ int rs8_lane(int q) { return ((q >> 2) & 1) | (q & 2) | ((q & 1) << 2); }
__device__ __forceinline__ double warp_rs8(const double (&v)[8], int lane) {
    const bool b0 = lane & 1, b1 = lane & 2, b2 = lane & 4;
    double a[4], c[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const double send = b0 ? v[i] : v[i + 4], keep = b0 ? v[i + 4] : v[i];
        a[i] = keep + __shfl_xor_sync(0xffffffffu, send, 1);
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const double send = b1 ? a[i] : a[i + 2], keep = b1 ? a[i + 2] : a[i];
        c[i] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    const double send = b2 ? c[0] : c[1], keep = b2 ? c[1] : c[0];
    double t = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    t += __shfl_xor_sync(0xffffffffu, t, 8);
    t += __shfl_xor_sync(0xffffffffu, t, 16);
    return t;
}

template <int CPW, int KR>
__global__ void __launch_bounds__(512, 1) k_qrcp_reg(int m, int Ng, double* __restrict__ Ag, int kmax, double eps,
                                                    int fixed, int* __restrict__ perm, double* __restrict__ rdiag,
                                                    int* __restrict__ out_nmu, long long* __restrict__ tprof) {
    static_assert(CPW <= 8, "reduce-scatter handles up to 8 columns per warp");
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double rsm2[];
    __shared__ QrSlot allslot[2][16];
    __shared__ double allx0[2][16];   // row j of each peer's candidate (pushed with the slot)
    __shared__ double s_wn2, s_x0;
    __shared__ int s_pos, s_rank, s_col, s_lc;
    __shared__ double wb_n2[16];      // per-warp best remaining column after each update
    __shared__ int wb_pos[16], wb_lc[16];
    const int CS = (int)cl.num_blocks(), b = (int)cl.block_rank(), tid = threadIdx.x;
    const int lane = tid & 31, warp = uniform_warp();
    constexpr int NW = 16;
    const int cpb = (Ng + CS - 1) / CS;
    const int c0 = b * cpb;
    const int nc = max(0, min(Ng, c0 + cpb) - c0);
    double* v = rsm2;                           // m (zero outside rows j..m-1)
    double* pub = v + m;                        // 2 x m published candidate copies
    double* n2 = pub + 2 * (size_t)m;           // cpb
    int* pos = reinterpret_cast<int*>(n2 + cpb);
    int* dn = pos + cpb;
    double col[CPW][KR];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int lc = warp + NW * q;
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int row = lane + 32 * k;
            col[q][k] = (lc < nc && row < m) ? Ag[(size_t)(c0 + lc) * m + row] : 0.0;
        }
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < KR; ++k) sq += col[q][k] * col[q][k];
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0 && lc < nc) {
            n2[lc] = sq;
            pos[lc] = c0 + lc;
            dn[lc] = 0;
        }
    }
    for (int i = tid; i < m; i += blockDim.x) v[i] = 0.0;
    __syncthreads();
    double r11 = 0.0;
    int N = kmax;
    cl.sync();
    for (int j = 0; j < kmax; ++j) {
        const int buf = j & 1;
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j] = clock64();
        if (warp == 0) {
            double bn = -1.0;
            int bp = 1 << 30, bl = -1;
            if (j == 0) {  // initial norms: scan the CTA's columns
                for (int lc = lane; lc < nc; lc += 32) {
                    const double xx = n2[lc];
                    if (xx > bn || (xx == bn && pos[lc] < bp)) {
                        bn = xx;
                        bp = pos[lc];
                        bl = lc;
                    }
                }
            } else if (lane < NW) {  // later steps: the warps' bests from the previous update
                bn = wb_n2[lane];
                bp = wb_pos[lane];
                bl = wb_lc[lane];
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bl = ol;
                }
            }
            if (lane == 0) s_lc = bl;
            if (lane < CS) {
                QrSlot sl;
                sl.n2 = bn;
                sl.pos = bp;
                sl.col = bl >= 0 ? c0 + bl : -1;
                cl.map_shared_rank(&allslot[0][0], lane)[buf * 16 + b] = sl;
            }
        }
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 1] = clock64();
        __syncthreads();
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 2] = clock64();
        {   // the owning warp publishes the candidate's rows j..m-1 from its registers and
            // pushes its row j to every peer next to the slot
            const int bl = s_lc;
            if (bl >= 0 && warp == bl % NW) {
                const int qs = bl / NW;
                double xj = 0.0;
#pragma unroll
                for (int q = 0; q < CPW; ++q)
                    if (q == qs)
#pragma unroll
                        for (int k = 0; k < KR; ++k) {
                            const int row = lane + 32 * k;
                            if (row >= j && row < m) pub[(size_t)buf * m + row] = col[q][k];
                            if (row == j) xj = col[q][k];
                        }
                xj = __shfl_sync(0xffffffffu, xj, j & 31);
                if (lane < CS) cl.map_shared_rank(&allx0[0][0], lane)[buf * 16 + b] = xj;
            }
        }
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 3] = clock64();
        cl.sync();
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 4] = clock64();
        if (warp == 0) {
            double bn = -1.0;
            int bp = 1 << 30, bs = -1, bc = -1;
            if (lane < CS) {
                const QrSlot sl = allslot[buf][lane];
                if (sl.col >= 0) {
                    bn = sl.n2;
                    bp = sl.pos;
                    bs = lane;
                    bc = sl.col;
                }
            }
            for (int o = 16; o > 0; o >>= 1) {
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int os = __shfl_xor_sync(0xffffffffu, bs, o);
                const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bs = os;
                    bc = oc;
                }
            }
            if (lane == 0) {
                s_wn2 = bn;
                s_pos = bp;
                s_rank = bs;
                s_col = bc;
                s_x0 = bs >= 0 ? allx0[buf][bs] : 0.0;
            }
        }
        __syncthreads();
        const double wn2 = s_wn2;
        const int pw = s_pos, ws = s_rank, cw = s_col;
        const double rjj = sqrt(fmax(wn2, 0.0));
        if (j == 0) r11 = rjj;
        if (__syncthreads_or(ws < 0 || rjj == 0.0 || (fixed <= 0 && rjj < eps * r11))) {
            N = j;
            break;
        }
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 5] = clock64();
        // winner's rows j..m-1 from its owner CTA (one DSMEM read per row, by one thread each)
        const double* x = cl.map_shared_rank(pub, ws) + (size_t)buf * m;
        const double x0 = s_x0;
        const double alpha = (x0 >= 0.0) ? -rjj : rjj;
        const double v0 = x0 - alpha;
        const double tau = 2.0 / (wn2 - x0 * x0 + v0 * v0);
        for (int i = j + tid; i < m; i += blockDim.x) v[i] = (i == j) ? v0 : x[i];
        if (j > 0 && tid == 0) v[j - 1] = 0.0;  // rows < j stay zero (cleared as j advances)
        if (b == 0 && tid == 0) rdiag[j] = rjj;
        __syncthreads();
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 6] = clock64();
        double vr[KR];
#pragma unroll
        for (int k = 0; k < KR; ++k) {
            const int row = lane + 32 * k;
            vr[k] = row < m ? v[row] : 0.0;
        }
        // all CPW columns of the warp at once (independent dot / shuffle / norm chains -> ILP)
        bool live[CPW];
        double d[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) d[q] = 0.0;
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
            const int lc = warp + NW * q;
            const bool valid = lc < nc;
            const bool piv = __all_sync(0xffffffffu, valid && c0 + lc == cw);
            live[q] = __all_sync(0xffffffffu, valid && !piv && dn[valid ? lc : 0] == 0);
            if (piv) {
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const int row = lane + 32 * k;
                    if (row == j) col[q][k] = alpha;
                    else if (row > j) col[q][k] = 0.0;
                }
                if (lane == 0) {
                    pos[lc] = j;
                    dn[lc] = 1;
                }
            }
#pragma unroll
            for (int k = 0; k < KR; ++k) d[q] += vr[k] * col[q][k];
        }
        // all CPW dot products in one reduce-scatter, then each lane fetches the totals
        const double dt = warp_rs8(d, lane);
        double nn[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) nn[q] = 0.0;
#pragma unroll
        for (int q = 0; q < CPW; ++q) {
            const double dq = __shfl_sync(0xffffffffu, dt, rs8_lane(q));
            if (live[q]) {
                const double f = tau * dq;
#pragma unroll
                for (int k = 0; k < KR; ++k) {
                    const double y = col[q][k] - f * vr[k];
                    col[q][k] = y;
                    if (lane + 32 * k > j) nn[q] += y * y;
                }
            }
        }
        const double nt = warp_rs8(nn, lane);
        {
            // lane l < 8 holds column q = rs8_index(l): store its norm and position (swap
            // semantics) and reduce the warp's best remaining column over lanes 0..7
            const int q = rs8_index(lane);
            bool lv = false;
#pragma unroll
            for (int qq = 0; qq < CPW; ++qq)
                if (qq == q) lv = live[qq];
            lv = lv && lane < 8;
            const int lc = warp + NW * q;
            double bn = -1.0;
            int bp = 1 << 30, bl = -1;
            if (lv) {
                int p = pos[lc];
                if (p == j) {
                    p = pw;
                    pos[lc] = pw;
                }
                n2[lc] = nt;
                bn = nt;
                bp = p;
                bl = lc;
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const double on = __shfl_xor_sync(0xffffffffu, bn, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
                if (on > bn || (on == bn && op < bp)) {
                    bn = on;
                    bp = op;
                    bl = ol;
                }
            }
            if (lane == 0) {
                wb_n2[warp] = bn;
                wb_pos[warp] = bp;
                wb_lc[warp] = bl;
            }
        }
        __syncthreads();
        if (tprof && b == 0 && tid == 0 && j < 512) tprof[8 * j + 7] = clock64();
    }
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
        const int lc = warp + NW * q;
        if (lc < nc)
#pragma unroll
            for (int k = 0; k < KR; ++k) {
                const int row = lane + 32 * k;
                if (row < m) Ag[(size_t)(c0 + lc) * m + row] = col[q][k];
            }
    }
    for (int lc = tid; lc < nc; lc += blockDim.x) perm[pos[lc]] = c0 + lc;
    if (b == 0 && tid == 0) *out_nmu = N;
    cl.sync();
}

// T = R11^{-1} R12 by column-oriented back substitution, one WARP per trailing column c (lane l
// keeps b_nu for nu = l, l+32, ... in registers), with R11 staged in shared memory (one CTA per
// SM, 32 warps, columns strided over the grid) and the reciprocals of its diagonal precomputed,
// so the per-column chain runs on shared-memory latency.  Used when N^2 doubles fit (N <= 160);
// larger N go through the blocked solve below.
template <int SLOTS>
__global__ void __launch_bounds__(1024) k_trsm_smem(int m, int Ng, int N, const double* __restrict__ A,
                                                   const int* __restrict__ perm, double* __restrict__ T) {
    extern __shared__ double rsm[];
    double* Rs = rsm;            // Rs[mu * N + nu] = R(nu, mu), nu <= mu
    double* rd = rsm + (size_t)N * N;
    for (int e = threadIdx.x; e < N * N; e += blockDim.x) {
        const int mu = e / N, nu = e - mu * N;
        Rs[e] = nu <= mu ? A[(size_t)perm[mu] * m + nu] : 0.0;
    }
    __syncthreads();
    for (int mu = threadIdx.x; mu < N; mu += blockDim.x) rd[mu] = 1.0 / Rs[(size_t)mu * N + mu];
    __syncthreads();
    const int l = threadIdx.x & 31;
    const int nwarps_total = gridDim.x * (blockDim.x >> 5);
    const int nc = Ng - N;
    for (int cc = blockIdx.x * (blockDim.x >> 5) + uniform_warp(); cc < nc; cc += nwarps_total) {
        const int c = N + cc;
        double b[SLOTS];
#pragma unroll
        for (int s = 0; s < SLOTS; ++s) {
            const int nu = s * 32 + l;
            b[s] = (nu < N) ? A[(size_t)perm[c] * m + nu] : 0.0;
        }
        for (int mu = N - 1; mu >= 0; --mu) {
            const int owner = mu & 31, slot = mu >> 5;
            double bm = 0.0;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s)
                if (s == slot) bm = b[s];
            double x = __shfl_sync(0xffffffffu, bm, owner) * rd[mu];
            if (l == owner) T[(size_t)mu * nc + cc] = x;
            const double* rcol = Rs + (size_t)mu * N;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int nu = s * 32 + l;
                if (nu < mu) b[s] -= rcol[nu] * x;
            }
        }
    }
}

// [R11 | R12] gathered contiguously (N x Ng, ld N; R11 upper triangle only) for the blocked solve.
__global__ void k_gather_R(int m, int Ng, int N, const double* __restrict__ A, const int* __restrict__ perm,
                           double* __restrict__ AB) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y + gridDim.y * blockIdx.z;
    if (i >= N || j >= Ng) return;
    AB[(size_t)j * N + i] = (j >= N || i <= j) ? A[(size_t)perm[j] * m + i] : 0.0;
}

// T = R11^{-1} R12.  Returns the strides of T(mu, c'): element at T[mu * tsm + c' * tsc].
static void trsm_cols(acp_context* ctx, int m, int Ng, int N, const double* A, const int* perm, double*& T,
                      size_t& tsm, size_t& tsc) {
    const int warps = Ng - N;
    tsm = (size_t)(Ng - N > 0 ? Ng - N : 1);
    tsc = 1;
    if (warps <= 0) return;
    const size_t smem = ((size_t)N * N + N) * sizeof(double);
    if (smem <= 200 * 1024) {
        int sms = 148;
        ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        const int blocks = std::min(sms, cdiv(warps, 32));
        auto launch = [&](auto kern) {
            func_attr((const void*)kern, 200 * 1024);
            kern<<<blocks, 1024, smem, ctx->stream>>>(m, Ng, N, A, perm, T);
        };
        if (N <= 64) launch(k_trsm_smem<2>);
        else if (N <= 128) launch(k_trsm_smem<4>);
        else launch(k_trsm_smem<8>);   // N^2 <= 25600 -> N <= 160
        launched(ctx);
        return;
    }
    // N > 160: gather [R11 | R12] and run the blocked upper-triangular solve (bsub + DMMA GEMM);
    // T is then column-major N x (Ng - N) inside the gathered array.
    double* AB = ctx->wsd("qr_RAB", (size_t)N * Ng);
    const int gz = cdiv(Ng, 65535);
    k_gather_R<<<dim3(cdiv(N, 128), cdiv(Ng, gz), gz), 128, 0, ctx->stream>>>(m, Ng, N, A, perm, AB);
    launched(ctx);
    upper_solve_blocked(ctx, AB, N, Ng - N);
    T = AB + (size_t)N * N;
    tsm = 1;
    tsc = (size_t)N;
}

// Xi[perm[c], mu] = T(mu, c - N) (c >= N) or delta_{c mu} (c < N);  S[mu] = perm[mu].
__global__ void k_scatter_xi(int Ng, int N, const int* __restrict__ perm, const double* __restrict__ T, size_t tsm,
                             size_t tsc, double* __restrict__ Xi, int* __restrict__ S) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    const int mu = blockIdx.y;
    if (c >= Ng) return;
    const int row = perm[c];
    double v;
    if (c < N) v = (c == mu) ? 1.0 : 0.0;
    else v = T[(size_t)mu * tsm + (size_t)(c - N) * tsc];
    Xi[(size_t)mu * Ng + row] = v;
    if (c == 0) S[mu] = perm[mu];
}

int compress(acp_context* ctx, const double* Psi, const double* Gp, int n_cols, const double* h_theta,
             const int* h_nu, int r_half, double id_eps, int n_fixed, int n_mu_max, int* S, double* Xi) {
    const int Ng = ctx->Ng;
    const int n_occ = ctx->sys.n_occ;
    ACP_REQUIRE(n_cols >= 1 && r_half >= 1 && r_half <= n_cols, "invalid sketch size");
    const int r = 2 * r_half;
    const int m = n_occ * r;
    // Omega from the raw draws
    double* d_theta = ctx->wsd("qr_theta", n_cols);
    int* d_nu = ctx->wsi("qr_nu", r_half);
    ACP_CUDA(cudaMemcpyAsync(d_theta, h_theta, n_cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ACP_CUDA(cudaMemcpyAsync(d_nu, h_nu, r_half * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    double* Om = ctx->wsd("qr_omega", (size_t)n_cols * r);
    k_srft_omega<<<dim3(cdiv(n_cols, 128), r_half), 128, 0, ctx->stream>>>(n_cols, r_half, d_theta, d_nu, Om);
    launched(ctx);
    double* Gt = ctx->wsd("qr_gt", (size_t)Ng * r);
    gemm_nn(ctx, Ng, n_cols, r, 1.0, Gp, Ng, Om, n_cols, 0.0, Gt, Ng);
    int kmax = m < Ng ? m : Ng;
    if (n_fixed > 0 && n_fixed < kmax) kmax = n_fixed;
    if (n_mu_max < kmax && n_fixed > 0) ACP_REQUIRE(false, "n_mu_fixed exceeds n_mu_max");
    // Large sketches (m > 256 rows, m N_g > 16M entries: configs[3], [4]): the structured QRCP
    // that never forms M~^T (qrcp_kron.cu); smaller ones (configs[2]: 7 vs 24 ms) keep the
    // formed-sketch kernels.  ACP_QRCP_KRON=1 / ACP_QRCP_DENSE=1 force either.
    const bool big = m > 256 && (size_t)m * Ng > ((size_t)16 << 20);
    if (kq_supported(r) && m > 64 && !getenv("ACP_QRCP_DENSE") && !getenv("ACP_QRCP_GRID") &&
        !getenv("ACP_QRCP_SMEM") && (big || getenv("ACP_QRCP_KRON"))) {
        // kmax <= n_mu_max: the columns of Q / R11 are sized by the caller's capacity
        return kq_compress(ctx, Psi, Gt, r, std::min(kmax, std::max(n_mu_max, 1) + (n_fixed > 0 ? 0 : 1)), id_eps,
                           n_fixed, n_mu_max, S, Xi);
    }
    // Kronecker rows
    double* A = ctx->wsd("qr_A", (size_t)m * Ng);
    {
        size_t smem = 32 * (size_t)(n_occ + r) * sizeof(double);
        func_attr((const void*)k_kron_rows, smem);
        k_kron_rows<<<cdiv(Ng, 32), 256, smem, ctx->stream>>>(Ng, n_occ, r, Psi, Gt, A);
        launched(ctx);
    }
    // QRCP: one persistent cooperative kernel
    int* perm = ctx->wsi("qr_perm", Ng);
    double* rdiag = ctx->wsd("qr_rdiag", m < Ng ? m : Ng);
    int* d_nmu = ctx->wsi("qr_nmu", 1);
    int dev_sms = 148;
    ACP_CUDA(cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device));
    // cluster path: the whole M~^T in the shared memory of <= 16 CTAs
    int csq = 0;
    size_t csmem = 0;
    for (int c = 1; c <= 16; c *= 2) {
        const int cpb = cdiv(Ng, c);
        const size_t bytes = ((size_t)cpb * m + 3 * (size_t)m + cpb) * sizeof(double) + 2 * (size_t)cpb * sizeof(int);
        if (bytes <= 200 * 1024 && cpb >= 1) {
            csq = c;
            csmem = bytes;
            // prefer a few CTAs over one: more SMs share the trailing updates
            if (c >= 4 || (size_t)Ng * m * sizeof(double) <= 64 * 1024) break;
        }
    }
    if (getenv("ACP_QRCP_GRID") || m > 256) csq = 0;  // test knob / register-resident update needs m <= 256
    // register-resident variant: (CPW, KR) = (8, 2) for m <= 64, (5, 8) for m <= 256
    int rcs = 0, rkind = 0;
    if (!getenv("ACP_QRCP_GRID") && !getenv("ACP_QRCP_SMEM")) {
        if (m <= 64 && cdiv(Ng, 16 * 8) <= 16) {
            rkind = 1;
            rcs = std::max(1, cdiv(Ng, 16 * 8));
        } else if (m <= 256 && cdiv(Ng, 16 * 5) <= 16) {
            rkind = 2;
            rcs = std::max(1, cdiv(Ng, 16 * 5));
        }
    }
    if (rkind) {
        auto kern = rkind == 1 ? k_qrcp_reg<8, 2> : k_qrcp_reg<5, 8>;
        const int cpb = cdiv(Ng, rcs);
        const size_t rsm = (3 * (size_t)m + cpb) * sizeof(double) + 2 * (size_t)cpb * sizeof(int);
        func_attr((const void*)kern, rsm, true);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(rcs, 1, 1);
        cfg.blockDim = dim3(512, 1, 1);
        cfg.dynamicSmemBytes = rsm;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = rcs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        long long* tprof = nullptr;
        const char* tpath = getenv("ACP_QR_PROFILE");
        if (tpath) {
            tprof = reinterpret_cast<long long*>(ctx->ws("qr_tprof", 8 * 512 * sizeof(long long)));
            ACP_CUDA(cudaMemsetAsync(tprof, 0, 8 * 512 * sizeof(long long), ctx->stream));
        }
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, m, Ng, A, kmax, id_eps, n_fixed, perm, rdiag, d_nmu, tprof));
        launched(ctx);
        if (tpath) {
            std::vector<long long> h(8 * 512);
            ACP_CUDA(cudaMemcpyAsync(h.data(), tprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            ACP_CUDA(cudaStreamSynchronize(ctx->stream));
            if (FILE* f = fopen(tpath, "a")) {
                for (int j = 0; j < 512 && h[8 * j]; ++j) {
                    for (int k = 0; k < 8; ++k) fprintf(f, "%lld ", h[8 * j + k]);
                    fprintf(f, "\n");
                }
                fclose(f);
            }
        }
        csq = -1;  // done
    }
    if (csq == -1) {
        // register-resident kernel already launched
    } else if (csq > 0) {
        auto kern = m <= 64 ? k_qrcp_cluster<2> : m <= 128 ? k_qrcp_cluster<4> : k_qrcp_cluster<8>;
        func_attr((const void*)kern, 200 * 1024, true);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(csq, 1, 1);
        cfg.blockDim = dim3(1024, 1, 1);
        cfg.dynamicSmemBytes = csmem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr1[1];
        attr1[0].id = cudaLaunchAttributeClusterDimension;
        attr1[0].val.clusterDim.x = csq;
        attr1[0].val.clusterDim.y = 1;
        attr1[0].val.clusterDim.z = 1;
        cfg.attrs = attr1;
        cfg.numAttrs = 1;
        long long* tprof = nullptr;
        const char* tpath = getenv("ACP_QR_PROFILE");
        if (tpath) {
            tprof = reinterpret_cast<long long*>(ctx->ws("qr_tprof", 8 * 512 * sizeof(long long)));
            ACP_CUDA(cudaMemsetAsync(tprof, 0, 8 * 512 * sizeof(long long), ctx->stream));
        }
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, m, Ng, A, kmax, id_eps, n_fixed, perm, rdiag, d_nmu, tprof));
        if (tpath) {
            std::vector<long long> h(8 * 512);
            ACP_CUDA(cudaMemcpyAsync(h.data(), tprof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost,
                                     ctx->stream));
            ACP_CUDA(cudaStreamSynchronize(ctx->stream));
            if (FILE* f = fopen(tpath, "a")) {
                for (int j = 0; j < 512 && h[8 * j]; ++j) {
                    for (int k = 0; k < 8; ++k) fprintf(f, "%lld ", h[8 * j + k]);
                    fprintf(f, "\n");
                }
                fclose(f);
            }
        }
        launched(ctx);
    } else {
        int G = dev_sms < Ng ? dev_sms : Ng;
        int cpb = cdiv(Ng, G);
        G = cdiv(Ng, cpb);
        const size_t tail = (size_t)m * sizeof(double) + (size_t)cpb * (sizeof(double) + 2 * sizeof(int)) + 64;
        const size_t smem_full = (size_t)cpb * m * sizeof(double) + tail;
        const bool use_smem = smem_full <= 200 * 1024 && !getenv("ACP_QRCP_NOSMEM");  // knob: tests
        const size_t smem = use_smem ? smem_full : tail;
        QrSlot* slots = static_cast<QrSlot*>(ctx->ws("qr_slots", 2 * (size_t)G * sizeof(QrSlot)));
        double* cand = ctx->wsd("qr_cand", 2 * (size_t)G * m);
        void* args[] = {(void*)&m, (void*)&Ng, (void*)&A, (void*)&kmax, (void*)&id_eps, (void*)&n_fixed,
                        (void*)&slots, (void*)&cand, (void*)&perm, (void*)&rdiag, (void*)&d_nmu};
        // global-memory columns: one warp per column, rows in registers, when m <= 2048
        int kr = (use_smem || getenv("ACP_QRCP_GRID16")) ? 0 : m <= 1024 ? 32 : m <= 2048 ? 64 : 1;
        if (kr == 1) kr = 2;      // two columns per warp (one column per warp: 20.9 vs 15.9 s per c4g step)
        if (!use_smem && getenv("ACP_QRCP_CHUNKED")) kr = 2;  // test knob: the chunked kernel at small m
        const void* fn = use_smem ? (const void*)k_qrcp_persistent<true, 0>
                         : kr == 1 ? (const void*)k_qrcp_persistent<false, 1>
                         : kr == 2 ? (const void*)k_qrcp_persistent<false, 2>
                         : kr == 32 ? (const void*)k_qrcp_persistent<false, 32>
                         : kr == 64 ? (const void*)k_qrcp_persistent<false, 64>
                                    : (const void*)k_qrcp_persistent<false, 0>;
        func_attr(fn, smem);
        int occ = 0;
        ACP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
        ACP_REQUIRE(occ >= 1 && G <= occ * dev_sms, "QRCP: cooperative grid does not fit");
        ACP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(256), args, smem, ctx->stream));
        launched(ctx);
    }
    int* hp = static_cast<int*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, d_nmu, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    const int N = *hp;
    ACP_REQUIRE(N >= 1, "QRCP selected no rows (zero sketch)");
    if (N > n_mu_max)
        throw Error(ACP_ERR_INVALID, "N_mu = " + std::to_string(N) + " exceeds n_mu_max = " + std::to_string(n_mu_max));
    // Xi
    double* T = ctx->wsd("qr_T", (size_t)N * (Ng - N > 0 ? Ng - N : 1));
    size_t tsm = 0, tsc = 0;
    trsm_cols(ctx, m, Ng, N, A, perm, T, tsm, tsc);
    k_scatter_xi<<<dim3(cdiv(Ng, 256), N), 256, 0, ctx->stream>>>(Ng, N, perm, T, tsm, tsc, Xi, S);
    launched(ctx);
    return N;
}


// ============================================================================ sharded QRCP
// Alg. 2 steps 2-3 with the N_g columns of M~^T split over ranks (one process
// per GPU): rank r owns grid points [col0, col0 + nloc).  One pivot step per launch:
//   (a) s > 0: every CTA selects the winner of step s-1 from the all-gathered candidates (largest
//       norm^2, lowest position on ties -- the same rule as the one-rank kernels), builds the
//       Householder vector from the winner's published column, records R11(:, s-1), swaps
//       positions s-1 <-> the winner's old position, updates the owned columns (exact norms);
//   (b) the rank's best remaining column (norm^2, position, index, all m rows) goes to `send`.
// The host all-gathers `send` (NCCL) into `recv` between launches.  The stop rule is decided
// identically by every CTA of every rank from the gathered data; after it, launches are no-ops.
struct QrsState {
    int stop;      // 1 once the rank threshold (or kmax) ended the factorisation
    int N;         // N_mu when stopped
    double r11;    // |R~_11|
};

__global__ void k_qrs_init(int m, int nloc, int col0, int Ng, int n_occ, int r, const double* __restrict__ Psi,
                           const double* __restrict__ Gt, double* __restrict__ A, int* __restrict__ pos,
                           int* __restrict__ dn, double* __restrict__ n2) {
    // one warp per owned column: its Kronecker row psi_i(a) G~(a, q) (row i + q n_occ) and norm^2
    const int lane = threadIdx.x & 31;
    const int lc = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (lc >= nloc) return;
    const int a = col0 + lc;
    double* c = A + (size_t)lc * m;
    double s = 0.0;
    for (int e = lane; e < m; e += 32) {
        const int i = e % n_occ, q = e / n_occ;
        const double v = Psi[(size_t)i * Ng + a] * Gt[(size_t)q * Ng + a];
        c[e] = v;
        s += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        n2[lc] = s;
        pos[lc] = a;
        dn[lc] = 0;
    }
}

template <int KR>
__global__ void __launch_bounds__(256) k_qrs_step(int m, int nloc, int col0, double* __restrict__ A, int s, int kmax,
                                                  const double* __restrict__ recv, int world, int stride, double eps,
                                                  int fixed, int* __restrict__ pos, int* __restrict__ dn,
                                                  double* __restrict__ n2, QrSlot* __restrict__ slots,
                                                  double* __restrict__ send, double* __restrict__ R11, int ldr,
                                                  int* __restrict__ piv, double* __restrict__ rdiag,
                                                  QrsState* __restrict__ st) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) double qsm[];
    __shared__ double red_d[32];
    __shared__ int red_i[32];
    __shared__ int red_j[32];
    const int G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    const int lane = tid & 31, warp = uniform_warp(), nwarp = blockDim.x >> 5;
    if (__ldcg(&st->stop)) return;  // set only by earlier launches: uniform
    const int cpb = (nloc + G - 1) / G;
    const int c0 = b * cpb;
    const int nc = max(0, min(nloc, c0 + cpb) - c0);
    double* v = qsm;
    if (s > 0) {
        const int j = s - 1;
        // ---- winner of step j among the gathered candidates (identical in every CTA and rank)
        double bn = -2.0;
        int bp = 1 << 30, bw = -1;
        for (int w = 0; w < world; ++w) {
            const double wn = recv[(size_t)w * stride];
            const int wp = (int)recv[(size_t)w * stride + 1];
            if (wn >= 0.0 && (wn > bn || (wn == bn && wp < bp))) {
                bn = wn;
                bp = wp;
                bw = w;
            }
        }
        const double rjj = bw >= 0 ? sqrt(fmax(bn, 0.0)) : 0.0;
        const double r11 = j == 0 ? rjj : __ldcg(&st->r11);
        if (bw < 0 || rjj == 0.0 || (fixed <= 0 && rjj < eps * r11)) {
            if (b == 0 && tid == 0) {
                st->stop = 1;
                st->N = j;
            }
            return;
        }
        const double* x = recv + (size_t)bw * stride + 3;
        const int cw = (int)recv[(size_t)bw * stride + 2];
        // ---- Householder vector from the published copy of the winner column
        double sx = 0.0;
        for (int i = j + tid; i < m; i += blockDim.x) {
            const double xi = x[i];
            v[i] = xi;
            sx += xi * xi;
        }
        for (int o = 16; o > 0; o >>= 1) sx += __shfl_xor_sync(0xffffffffu, sx, o);
        if (lane == 0) red_d[warp] = sx;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < nwarp; ++w) t += red_d[w];
            red_d[0] = t;
        }
        __syncthreads();
        const double xn2 = red_d[0];
        const double xn = sqrt(xn2);
        const double x0 = v[j];
        const double alpha = (x0 >= 0.0) ? -xn : xn;
        const double v0 = x0 - alpha;
        const double tau = 2.0 / (xn2 - x0 * x0 + v0 * v0);
        __syncthreads();
        if (tid == 0) v[j] = v0;
        if (b == 0) {
            for (int i = tid; i < j; i += blockDim.x) R11[(size_t)j * ldr + i] = x[i];
            if (tid == 0) {
                R11[(size_t)j * ldr + j] = alpha;
                piv[j] = cw;
                rdiag[j] = xn;
                if (j == 0) st->r11 = rjj;
            }
        }
        // ---- position bookkeeping (swap of positions j and bp) for the owned columns
        for (int lc = tid; lc < nc; lc += blockDim.x) {
            const int g = c0 + lc;
            if (col0 + g == cw) {
                pos[g] = j;
                dn[g] = 1;
            } else if (!dn[g] && pos[g] == j) {
                pos[g] = bp;
            }
        }
        __syncthreads();
        auto colp = [&](int lc) -> double* { return A + (size_t)(c0 + lc) * m; };
        if constexpr (KR == 32)
            qr_update_cols_warp<32>(colp, warp, nc, col0 + c0, cw, j, m, alpha, tau, v, dn + c0, n2 + c0);
        else if constexpr (KR == 64)
            qr_update_cols_warp1<64>(colp, warp, nc, col0 + c0, cw, j, m, alpha, tau, v, dn + c0, n2 + c0);
        else
            qr_update_cols_chunked2<16>(colp, warp, nc, col0 + c0, cw, j, m, alpha, tau, v, dn + c0, n2 + c0);
        __threadfence();
        grid.sync();
    }
    if (s >= kmax) {
        if (b == 0 && tid == 0) {
            st->stop = 1;
            st->N = s;
        }
        return;
    }
    // ---- (b) this CTA's best remaining column, then the rank's best (CTA 0) -> send
    if (warp == 0) {
        double bn = -1.0;
        int bp = 1 << 30, bl = -1;
        for (int lc = lane; lc < nc; lc += 32) {
            if (dn[c0 + lc]) continue;
            const double xv = __ldcg(&n2[c0 + lc]);
            const int pv = pos[c0 + lc];
            if (xv > bn || (xv == bn && pv < bp)) {
                bn = xv;
                bp = pv;
                bl = lc;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double on = __shfl_xor_sync(0xffffffffu, bn, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            const int ol = __shfl_xor_sync(0xffffffffu, bl, o);
            if (on > bn || (on == bn && op < bp)) {
                bn = on;
                bp = op;
                bl = ol;
            }
        }
        if (lane == 0) {
            QrSlot sl;
            sl.n2 = bn;
            sl.pos = bp;
            sl.col = bl >= 0 ? c0 + bl : -1;  // local column index
            slots[b] = sl;
        }
    }
    __threadfence();
    grid.sync();
    if (b != 0) return;
    double bn = -1.0;
    int bp = 1 << 30, bc = -1;
    for (int q = tid; q < G; q += blockDim.x) {
        const double sn = __ldcg(&slots[q].n2);
        const int sp = __ldcg(&slots[q].pos);
        const int sc = __ldcg(&slots[q].col);
        if (sc >= 0 && (sn > bn || (sn == bn && sp < bp))) {
            bn = sn;
            bp = sp;
            bc = sc;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double on = __shfl_xor_sync(0xffffffffu, bn, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (oc >= 0 && (bc < 0 || on > bn || (on == bn && op < bp))) {
            bn = on;
            bp = op;
            bc = oc;
        }
    }
    if (lane == 0) {
        red_d[warp] = bn;
        red_i[warp] = bp;
        red_j[warp] = bc;
    }
    __syncthreads();
    if (tid == 0) {
        for (int w = 1; w < nwarp; ++w)
            if (red_j[w] >= 0 && (red_j[0] < 0 || red_d[w] > red_d[0] || (red_d[w] == red_d[0] && red_i[w] < red_i[0]))) {
                red_d[0] = red_d[w];
                red_i[0] = red_i[w];
                red_j[0] = red_j[w];
            }
        send[0] = red_j[0] >= 0 ? red_d[0] : -1.0;
        send[1] = (double)red_i[0];
        send[2] = (double)(red_j[0] >= 0 ? col0 + red_j[0] : -1);
    }
    __syncthreads();
    const int lcw = red_j[0];
    if (lcw >= 0) {
        const double* c = A + (size_t)lcw * m;
        for (int i = tid; i < m; i += blockDim.x) send[3 + i] = __ldcg(&c[i]);
    }
}

// After the stop: Xi^T rows of the owned grid points, XiT[lc * N + mu] = (R11^{-1} R(0:N, a))_mu for
// a non-pivot column a = col0 + lc, delta(mu, position) for a pivot.
__global__ void k_qrs_gather(int m, int nloc, int N, const double* __restrict__ A, const double* __restrict__ R11,
                             int ldr, double* __restrict__ AB) {
    // AB = [R11 | R(0:N, owned)] column-major, ld N
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int jc = blockIdx.y + gridDim.y * blockIdx.z;
    if (i >= N || jc >= N + nloc) return;
    AB[(size_t)jc * N + i] = jc < N ? (i <= jc ? R11[(size_t)jc * ldr + i] : 0.0) : A[(size_t)(jc - N) * m + i];
}

__global__ void k_qrs_xi(int nloc, int N, const double* __restrict__ T, const int* __restrict__ pos,
                         const int* __restrict__ dn, double* __restrict__ XiT) {
    const int mu = blockIdx.x * blockDim.x + threadIdx.x;
    const int lc = blockIdx.y + gridDim.y * blockIdx.z;
    if (mu >= N || lc >= nloc) return;
    const bool pv = dn[lc] && pos[lc] < N;
    XiT[(size_t)lc * N + mu] = pv ? (pos[lc] == mu ? 1.0 : 0.0) : T[(size_t)lc * N + mu];
}

int qrs_begin(acp_context* ctx, const double* Psi, const double* Gp, int n_cols, const double* h_theta,
              const int* h_nu, int r_half, int col_begin, int col_end, int n_fixed, int n_mu_max) {
    const int Ng = ctx->Ng, n_occ = ctx->sys.n_occ;
    ACP_REQUIRE(n_cols >= 1 && r_half >= 1 && r_half <= n_cols, "invalid sketch size");
    ACP_REQUIRE(0 <= col_begin && col_begin <= col_end && col_end <= Ng, "invalid column range");
    const int r = 2 * r_half, m = n_occ * r, nloc = col_end - col_begin;
    double* d_theta = ctx->wsd("qr_theta", n_cols);
    int* d_nu = ctx->wsi("qr_nu", r_half);
    ACP_CUDA(cudaMemcpyAsync(d_theta, h_theta, n_cols * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    ACP_CUDA(cudaMemcpyAsync(d_nu, h_nu, r_half * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
    double* Om = ctx->wsd("qr_omega", (size_t)n_cols * r);
    k_srft_omega<<<dim3(cdiv(n_cols, 128), r_half), 128, 0, ctx->stream>>>(n_cols, r_half, d_theta, d_nu, Om);
    launched(ctx);
    double* Gt = ctx->wsd("qr_gt", (size_t)Ng * r);
    gemm_nn(ctx, Ng, n_cols, r, 1.0, Gp, Ng, Om, n_cols, 0.0, Gt, Ng);
    int kmax = std::min(m, Ng);
    if (n_fixed > 0) kmax = std::min(kmax, n_fixed);
    kmax = std::min(kmax, n_mu_max);
    const int nl = std::max(nloc, 1);
    double* A = ctx->wsd("qrs_A", (size_t)m * nl);
    int* pos = ctx->wsi("qrs_pos", nl);
    int* dn = ctx->wsi("qrs_dn", nl);
    double* n2 = ctx->wsd("qrs_n2", nl);
    ctx->wsd("qrs_R11", (size_t)kmax * kmax);
    ctx->wsi("qrs_piv", kmax);
    ctx->wsd("qrs_rdiag", kmax);
    QrsState* st = static_cast<QrsState*>(ctx->ws("qrs_state", sizeof(QrsState)));
    ACP_CUDA(cudaMemsetAsync(st, 0, sizeof(QrsState), ctx->stream));
    if (nloc > 0) {
        k_qrs_init<<<cdiv(nloc, 8), 256, 0, ctx->stream>>>(m, nloc, col_begin, Ng, n_occ, r, Psi, Gt, A, pos, dn, n2);
        launched(ctx);
    }
    ctx->qrs_m = m;
    ctx->qrs_kmax = kmax;
    ctx->qrs_col0 = col_begin;
    ctx->qrs_nloc = nloc;
    ctx->qrs_fixed = n_fixed;
    return m;
}

void qrs_step(acp_context* ctx, int s, const double* recv, int world, double id_eps, double* send) {
    const int m = ctx->qrs_m, nloc = ctx->qrs_nloc, kmax = ctx->qrs_kmax, col0 = ctx->qrs_col0;
    double* A = ctx->wsd("qrs_A", (size_t)m * std::max(nloc, 1));
    int* pos = ctx->wsi("qrs_pos", std::max(nloc, 1));
    int* dn = ctx->wsi("qrs_dn", std::max(nloc, 1));
    double* n2 = ctx->wsd("qrs_n2", std::max(nloc, 1));
    double* R11 = ctx->wsd("qrs_R11", (size_t)kmax * kmax);
    int* piv = ctx->wsi("qrs_piv", kmax);
    double* rdiag = ctx->wsd("qrs_rdiag", kmax);
    QrsState* st = static_cast<QrsState*>(ctx->ws("qrs_state", sizeof(QrsState)));
    int sms = 148;
    ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    int G = std::max(1, std::min(sms, cdiv(std::max(nloc, 1), 8)));
    QrSlot* slots = static_cast<QrSlot*>(ctx->ws("qrs_slots", (size_t)sms * sizeof(QrSlot)));
    const int stride = m + 3;
    int fixed = ctx->qrs_fixed;
    double eps = id_eps;
    int ldr = kmax;
    const size_t smem = (size_t)m * sizeof(double);
    const void* fn = m <= 1024 ? (const void*)k_qrs_step<32> : m <= 2048 ? (const void*)k_qrs_step<64>
                                                                          : (const void*)k_qrs_step<0>;
    func_attr(fn, smem);
    int occ = 0;
    ACP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
    ACP_REQUIRE(occ >= 1, "sharded QRCP: kernel does not fit");
    G = std::min(G, occ * sms);
    void* args[] = {(void*)&m, (void*)&nloc, (void*)&col0, (void*)&A, (void*)&s, (void*)&kmax, (void*)&recv,
                    (void*)&world, (void*)&stride, (void*)&eps, (void*)&fixed, (void*)&pos, (void*)&dn, (void*)&n2,
                    (void*)&slots, (void*)&send, (void*)&R11, (void*)&ldr, (void*)&piv, (void*)&rdiag, (void*)&st};
    ACP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(256), args, smem, ctx->stream));
    launched(ctx);
}

void qrs_status(acp_context* ctx, int* stop, int* N) {
    QrsState* st = static_cast<QrsState*>(ctx->ws("qrs_state", sizeof(QrsState)));
    QrsState* hp = static_cast<QrsState*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, st, sizeof(QrsState), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    *stop = hp->stop;
    *N = hp->N;
}

int qrs_finish(acp_context* ctx, int* S, double* XiT) {
    int stop = 0, N = 0;
    qrs_status(ctx, &stop, &N);
    ACP_REQUIRE(stop, "sharded QRCP: finish before the factorisation stopped");
    ACP_REQUIRE(N >= 1, "QRCP selected no rows (zero sketch)");
    const int m = ctx->qrs_m, nloc = ctx->qrs_nloc, kmax = ctx->qrs_kmax;
    const double* A = ctx->wsd("qrs_A", (size_t)m * std::max(nloc, 1));
    const int* pos = ctx->wsi("qrs_pos", std::max(nloc, 1));
    const int* dn = ctx->wsi("qrs_dn", std::max(nloc, 1));
    const double* R11 = ctx->wsd("qrs_R11", (size_t)kmax * kmax);
    const int* piv = ctx->wsi("qrs_piv", kmax);
    ACP_CUDA(cudaMemcpyAsync(S, piv, N * sizeof(int), cudaMemcpyDeviceToDevice, ctx->stream));
    if (nloc == 0) return N;
    double* AB = ctx->wsd("qrs_AB", (size_t)N * (N + nloc));
    const int ncol = N + nloc, gz = cdiv(ncol, 65535);
    k_qrs_gather<<<dim3(cdiv(N, 128), cdiv(ncol, gz), gz), 128, 0, ctx->stream>>>(m, nloc, N, A, R11, kmax, AB);
    launched(ctx);
    upper_solve_blocked(ctx, AB, N, nloc);
    const int gz2 = cdiv(nloc, 65535);
    k_qrs_xi<<<dim3(cdiv(N, 128), cdiv(nloc, gz2), gz2), 128, 0, ctx->stream>>>(nloc, N, AB + (size_t)N * N, pos, dn,
                                                                                 XiT);
    launched(ctx);
    return N;
}

}  // namespace acp
