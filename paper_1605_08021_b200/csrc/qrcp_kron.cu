// qrcp_kron.cu -- column-pivoted QR of the Kronecker sketch M~^T without forming it (Alg. 2 steps
// 2-4), for the large sketches (configs[2..4]).
//
// Column a of M~^T is psi(a) (x) g~(a) (row i + q N_occ = psi_i(a) G~(a, q)), so
// M~^T never needs to exist: with Q_j = [q_0 .. q_{j-1}] the orthonormal factor so far,
//   R(j, a)   = q_j^T (psi(a) (x) g~(a)) = sum_q G~(a, q) sum_i psi_i(a) q_j[i + q N_occ]
// is one pass over Psi (N_g x N_occ) per pivot, and the trailing column norms are DOWNDATED,
// n2(a) -= R(j, a)^2.  Downdating loses accuracy (~ j eps |a|^2) where a column's norm has
// dropped a lot, so n2 only SCREENS: every column within 64 eps (j+1) max|a|^2 of the largest n2
// is a candidate, and for each candidate the trailing component y_c = (I - Q_j Q_j^T) a_c and its
// EXACT norm are formed; the winner is the candidate with the largest exact norm (lowest current
// position on ties) -- the greedy rule of the oracle (reading R8), decided on exact trailing
// norms.  The winner's component is re-orthogonalised once (CGS2) and becomes q_j; R11(:, j) =
// Q_j^T a_w, R(j, j) = |y'_w|.  The stop rule is the oracle's: |R_jj| < eps |R_11|.
// The candidates' coefficients Q_j^T a_c are columns of the R rows already computed (R(k, a) for
// every grid point a at every pivot k), so per pivot: one pass over Psi and three over Q_j (m x j)
// -- instead of a read and a write of the whole m x N_g sketch per pivot (k_qrcp_persistent).  ONE cooperative launch, grid barriers
// between the phases; every reduction has a fixed order.
#include <cooperative_groups.h>
#include <cstdio>

#include "common.cuh"

namespace acp {

namespace cgk = cooperative_groups;

constexpr int KQ_CMAX = 16;  // candidates verified per pivot
constexpr int KQ_T = 256;
constexpr int KQ_U = 16;   // loads in flight per thread in the passes over Q
constexpr int KQ_UP = 32;  // psi fragments in flight per lane in the R-row DMMA pass

struct KqArgs {
    int m, Ng, n_occ, r, kmax, fixed;
    double eps;
    const double* Psi;   // (n_occ, Ng): psi_i(a) at Psi[i Ng + a]
    const double* Gt;    // (Ng, r) column-major: G~(a, q) at Gt[q Ng + a]
    double* Q;           // m x kmax column-major
    double* Rrows;       // kmax x Ng: R(j, a) at Rrows[j Ng + a]
    double* R11;         // kmax x kmax column-major (upper)
    double* n2;          // Ng: downdated trailing norm^2
    int* pos;            // Ng: current position (swap semantics)
    int* dn;             // Ng: pivoted flag
    int* piv;            // kmax: pivot grid index per step
    double* rdiag;       // kmax
    double* slots;       // G: per-CTA max n2
    double* tpart;       // G x CMAX: per-CTA partial exact norms
    double* Y;           // CMAX x m: candidate components (y_c)
    double* w2;          // kmax: Q^T y_w (second pass)
    int* cand;           // 2 x CMAX
    int* ncand;          // 2
    int* out_nmu;
    int* overflow;       // set when more than CMAX columns were within the screening window
    long long* prof;     // debug (ACP_KQ_PROF): CTA 0's cycles per phase, summed over pivots, or null
    int psi_keep;        // grid points a < psi_keep: Psi loads marked L2 evict_last, the rest evict_first
    int q_last;          // 1: the passes over Q mark their loads L2 evict_last
};

#define KQ_MARK(ph)                                                          \
    do {                                                                     \
        if (g.prof && b == 0 && t == 0) {                                    \
            const long long now_ = clock64();                                \
            g.prof[ph] += now_ - tmark;                                      \
            tmark = now_;                                                    \
        }                                                                    \
    } while (0)

__device__ __forceinline__ void dmma_kq(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// Psi (N_g x N_occ, 134 MB at c4g) does not fit the 126 MB L2 and is streamed in the same order
// every pivot: its loads carry an L2 policy (a share of the grid points may be pinned evict_last,
// the rest streams evict_first) so that it does not flush Q from L2.
__device__ __forceinline__ unsigned long long kq_pol(bool keep) {
    unsigned long long p;
    if (keep) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double kq_ld_ro(const double* a, unsigned long long pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
// Q is written by the kernel itself: L2-only (cg) loads, optionally with a cache hint
__device__ __forceinline__ double kq_ld_q(const double* a, bool hint, unsigned long long pol) {
    if (!hint) return __ldcg(a);
    double v;
    asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

__device__ __forceinline__ double kq_warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void k_kq_init(int Ng, int n_occ, int r, const double* __restrict__ Psi, const double* __restrict__ Gt,
                          double* __restrict__ n2, int* __restrict__ pos, int* __restrict__ dn) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= Ng) return;
    double sp = 0.0, sg = 0.0;
    for (int i = 0; i < n_occ; ++i) {
        const double v = Psi[(size_t)i * Ng + a];
        sp += v * v;
    }
    for (int q = 0; q < r; ++q) {
        const double v = Gt[(size_t)q * Ng + a];
        sg += v * v;
    }
    n2[a] = sp * sg;  // |psi(a) (x) g~(a)|^2
    pos[a] = a;
    dn[a] = 0;
}

template <int RQ>
__global__ void __launch_bounds__(KQ_T, 2) k_kq(KqArgs g) {
    cgk::grid_group grid = cgk::this_grid();
    extern __shared__ __align__(16) double ksm[];
    __shared__ double red[KQ_T / 32];
    __shared__ double sred[KQ_T / 32][KQ_CMAX];
    __shared__ int s_int[4];
    const int G = gridDim.x, b = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int nwarp = KQ_T / 32, GW = G * nwarp, gw = b * nwarp + warp;
    const int m = g.m, Ng = g.Ng, n_occ = g.n_occ;
    const int apb = (Ng + G - 1) / G, a0 = b * apb, a1 = min(Ng, a0 + apb);   // owned grid points
    const int epb = (m + G - 1) / G, e0 = b * epb, e1 = min(m, e0 + epb);     // owned sketch rows
    double* cps = ksm;                          // CMAX x n_occ  candidate psi(c)
    double* cgs = cps + KQ_CMAX * n_occ;        // CMAX x RQ     candidate g~(c)
    double* qs = cgs + KQ_CMAX * RQ;            // m             q_j for the R-row pass
    double maxn0 = 0.0, r11 = 0.0;
    int N = g.kmax;
    long long tmark = (g.prof && b == 0 && t == 0) ? clock64() : 0;
    const unsigned long long pkeep = kq_pol(true), pstream = kq_pol(false);
    const bool qh = g.q_last != 0;
    // P1: per-CTA max of the screening norms (for pivot jn; also resets the candidate counter
    // pivot jn + 1 will use -- nobody touches it before then).  Run once here and then at the end
    // of every pivot's R-row pass, so it shares that pass's grid barrier.
    auto p1 = [&](int jn) {
        double mx = -1.0;
        for (int a = a0 + t; a < a1; a += KQ_T)
            if (!g.dn[a]) mx = fmax(mx, g.n2[a]);
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) red[warp] = mx;
        __syncthreads();
        if (t == 0) {
            double v = red[0];
            for (int w = 1; w < nwarp; ++w) v = fmax(v, red[w]);
            g.slots[b] = v;
            if (b == 0) g.ncand[(jn & 1) ^ 1] = 0;
        }
        __syncthreads();
    };
    p1(0);
    __threadfence();
    grid.sync();
    for (int j = 0; j < g.kmax; ++j) {
        const int par = j & 1;
        KQ_MARK(0);
        // ---- P2: global max, screening window, candidate list
        double M = -1.0;
        for (int q = t; q < G; q += KQ_T) M = fmax(M, __ldcg(&g.slots[q]));
        for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
        if (lane == 0) red[warp] = M;
        __syncthreads();
        M = red[0];
        for (int w = 1; w < nwarp; ++w) M = fmax(M, red[w]);
        __syncthreads();
        if (j == 0) maxn0 = M;
        if (M <= 0.0) {  // nothing left (zero sketch or every column taken)
            N = j;
            break;
        }
        const double thr = M - 64.0 * 1.1102230246251565e-16 * (double)(j + 1) * maxn0;
        for (int a = a0 + t; a < a1; a += KQ_T) {
            if (!g.dn[a] && g.n2[a] >= thr) {
                const int k = atomicAdd(&g.ncand[par], 1);
                if (k < KQ_CMAX) g.cand[par * KQ_CMAX + k] = a;
                else g.overflow[0] = 1;
            }
        }
        __threadfence();
        grid.sync();
        KQ_MARK(1);
        // ---- P3: the candidates' psi(c), g~(c) staged in shared memory.  Their coefficients in the
        // current basis, W(k, c) = q_k^T a_c (k < j), are the R rows the earlier pivots' P6 passes
        // already produced for every grid point: W(k, c) = R(k, c) = Rrows[k Ng + c] (no pass over Q)
        const int nc = min(__ldcg(&g.ncand[par]), KQ_CMAX);
        for (int e = t; e < nc * n_occ; e += KQ_T) {
            const int c = e / n_occ, i = e - c * n_occ;
            cps[e] = g.Psi[(size_t)i * Ng + __ldcg(&g.cand[par * KQ_CMAX + c])];
        }
        for (int e = t; e < nc * RQ; e += KQ_T) {
            const int c = e / RQ, q = e - c * RQ;
            cgs[e] = g.Gt[(size_t)q * Ng + __ldcg(&g.cand[par * KQ_CMAX + c])];
        }
        __syncthreads();
        KQ_MARK(2);
        // ---- P4: y_c = a_c - Q W(:, c) on the owned rows, exact norms (per-CTA partials)
        {
            const int nrow = e1 - e0;
            // threads: (row, k-slice); the slices are summed in shared memory in slice order
            const int slices = nrow > 0 ? max(1, KQ_T / nrow) : 1;
            double* sacc = qs;  // scratch: slices x nrow
            const int rr = t % max(nrow, 1), sl = t / max(nrow, 1);
            for (int c = 0; c < nc; ++c) {
                const int ac = __ldcg(&g.cand[par * KQ_CMAX + c]);
                if (nrow > 0 && sl < slices) {
                    const int e = e0 + rr;
                    double s = 0.0;
                    for (int kb = sl; kb < j; kb += KQ_U * slices) {
                        double qv[KQ_U], wv[KQ_U];
#pragma unroll
                        for (int u = 0; u < KQ_U; ++u) {  // eight independent load pairs in flight
                            const int k = kb + u * slices;
                            qv[u] = k < j ? kq_ld_q(&g.Q[(size_t)k * m + e], qh, pkeep) : 0.0;
                            wv[u] = k < j ? __ldcg(&g.Rrows[(size_t)k * Ng + ac]) : 0.0;
                        }
#pragma unroll
                        for (int u = 0; u < KQ_U; ++u) s += qv[u] * wv[u];
                    }
                    sacc[sl * nrow + rr] = s;
                }
                __syncthreads();
                double y2 = 0.0;
                if (t < nrow) {
                    const int e = e0 + t;
                    double s = 0.0;
                    for (int q = 0; q < slices; ++q) s += sacc[q * nrow + t];
                    const int qi = e / n_occ, i = e - qi * n_occ;
                    const double y = cps[c * n_occ + i] * cgs[c * RQ + qi] - s;
                    g.Y[(size_t)c * m + e] = y;
                    y2 = y * y;
                }
                y2 = kq_warp_sum(y2);
                if (lane == 0) sred[warp][c] = y2;
                __syncthreads();
            }
            if (t < nc) {
                double s = 0.0;
                for (int w = 0; w < nwarp; ++w) s += sred[w][t];
                g.tpart[(size_t)b * KQ_CMAX + t] = s;
            }
        }
        __threadfence();
        grid.sync();
        KQ_MARK(3);
        // ---- P5: the winner (largest exact norm, lowest position), stop rule, CGS2 second pass
        {
            // exact norms: thread (slice sl, candidate c) sums every 16th CTA partial; the 16 slices
            // are then added in slice order (fixed order, all loads in flight at once)
            const int c = t & 15, sl = t >> 4;
            double tc = 0.0;
            if (c < nc)
                for (int q = sl; q < G; q += 16) tc += __ldcg(&g.tpart[(size_t)q * KQ_CMAX + c]);
            qs[sl * 16 + c] = tc;  // qs (free after P4) as a [16][16] scratch
            __syncthreads();
            if (t < KQ_CMAX) {
                double v = -1.0;
                if (t < nc) {
                    v = 0.0;
                    for (int q = 0; q < 16; ++q) v += qs[q * 16 + t];
                }
                sred[0][t] = v;
            }
        }
        __syncthreads();
        if (t == 0) {
            int bc = -1;
            double bt = -1.0;
            int bp = 1 << 30;
            for (int c = 0; c < nc; ++c) {
                const int a = __ldcg(&g.cand[par * KQ_CMAX + c]);
                const double tc = sred[0][c];
                const int pc = __ldcg(&g.pos[a]);
                if (tc > bt || (tc == bt && pc < bp)) {
                    bt = tc;
                    bp = pc;
                    bc = c;
                }
            }
            s_int[0] = bc;
            s_int[1] = bp;
            red[0] = bt;
        }
        __syncthreads();
        const int wc = s_int[0];
        const double tw = red[0];
        const double rjj = sqrt(fmax(tw, 0.0));
        if (j == 0) r11 = rjj;
        if (wc < 0 || rjj == 0.0 || (g.fixed <= 0 && rjj < g.eps * r11)) {
            N = j;
            break;
        }
        const int aw = __ldcg(&g.cand[par * KQ_CMAX + wc]);
        const double* yw = g.Y + (size_t)wc * m;
        // w2 = Q^T y_w
        for (int k = gw; k < j; k += GW) {
            const double* qk = g.Q + (size_t)k * m;
            double s = 0.0;
            for (int e0b = 0; e0b < m; e0b += 32 * KQ_U) {
                double qv[KQ_U], yv[KQ_U];
#pragma unroll
                for (int u = 0; u < KQ_U; ++u) {
                    const int e = e0b + lane + 32 * u;
                    qv[u] = e < m ? kq_ld_q(&qk[e], qh, pkeep) : 0.0;
                    yv[u] = e < m ? __ldcg(&yw[e]) : 0.0;
                }
#pragma unroll
                for (int u = 0; u < KQ_U; ++u) s += qv[u] * yv[u];
            }
            s = kq_warp_sum(s);
            if (lane == 0) g.w2[k] = s;
        }
        __threadfence();
        grid.sync();
        KQ_MARK(4);
        // y' = y_w - Q w2 on the owned rows (kept in shared memory), norm partials
        {
            const int nrow = e1 - e0;
            const int slices = nrow > 0 ? max(1, KQ_T / nrow) : 1;
            double* sacc = qs;
            const int rr = t % max(nrow, 1), sl = t / max(nrow, 1);
            if (nrow > 0 && sl < slices) {
                const int e = e0 + rr;
                double s = 0.0;
                for (int kb = sl; kb < j; kb += KQ_U * slices) {
                    double qv[KQ_U], wv[KQ_U];
#pragma unroll
                    for (int u = 0; u < KQ_U; ++u) {
                        const int k = kb + u * slices;
                        qv[u] = k < j ? kq_ld_q(&g.Q[(size_t)k * m + e], qh, pkeep) : 0.0;
                        wv[u] = k < j ? __ldcg(&g.w2[k]) : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < KQ_U; ++u) s += qv[u] * wv[u];
                }
                sacc[sl * nrow + rr] = s;
            }
            __syncthreads();
            double yv = 0.0;
            if (t < nrow) {
                double s = 0.0;
                for (int q = 0; q < slices; ++q) s += sacc[q * nrow + t];
                yv = __ldcg(&yw[e0 + t]) - s;
            }
            __syncthreads();
            if (t < nrow) sacc[t] = yv;  // keep y' of the owned rows
            const double s = kq_warp_sum(yv * yv);
            if (lane == 0) red[warp] = s;
            __syncthreads();
            if (t == 0) {
                double v = 0.0;
                for (int w = 0; w < nwarp; ++w) v += red[w];
                g.tpart[(size_t)b * KQ_CMAX] = v;
            }
        }
        __threadfence();
        grid.sync();
        KQ_MARK(5);
        {
            double nn = 0.0;
            for (int q = t; q < G; q += KQ_T) nn += __ldcg(&g.tpart[(size_t)q * KQ_CMAX]);
            nn = kq_warp_sum(nn);
            if (lane == 0) red[warp] = nn;
            __syncthreads();
            nn = 0.0;
            for (int w = 0; w < nwarp; ++w) nn += red[w];
            const double nrm = sqrt(nn);
            const int nrow = e1 - e0;
            if (t < nrow) g.Q[(size_t)j * m + e0 + t] = qs[t] / nrm;
            // R11(:, j) = Q^T a_w (first pass + correction), spread over all CTAs
            for (int k = b * KQ_T + t; k < j; k += G * KQ_T)
                g.R11[(size_t)j * g.kmax + k] = __ldcg(&g.Rrows[(size_t)k * Ng + aw]) + __ldcg(&g.w2[k]);
            if (b == 0 && t == 0) {
                g.R11[(size_t)j * g.kmax + j] = nrm;
                g.piv[j] = aw;
                g.rdiag[j] = nrm;
            }
            // position bookkeeping: the winner takes position j, the column at j takes its old one
            const int pw = s_int[1];
            for (int a = a0 + t; a < a1; a += KQ_T) {
                if (a == aw) {
                    g.pos[a] = j;
                    g.dn[a] = 1;
                } else if (!g.dn[a] && g.pos[a] == j) {
                    g.pos[a] = pw;
                }
            }
        }
        __threadfence();
        grid.sync();
        KQ_MARK(6);
        // ---- P6: R(j, a) for every grid point (one pass over Psi), downdate the screening norms
        // q_j staged as [q][i] with row stride n_occ + 4: the B fragments of a warp (i = i0 + lane % 4,
        // q = lane / 4) then hit 32 distinct banks
        for (int e = t; e < m; e += KQ_T) {
            const int q = e / n_occ, i = e - q * n_occ;
            qs[i + q * (n_occ + 4)] = __ldcg(&g.Q[(size_t)j * m + e]);
        }
        __syncthreads();
        // P(a, q) = sum_i psi_i(a) Q3(i, q) as FP64 DMMA tiles (mma.sync m8n8k4: 8 grid points x 8
        // sketch columns x 4 orbitals; A = psi rows straight from global memory, B = q_j from shared
        // memory), then R(j, a) = sum_q G~(a, q) P(a, q) across the four lanes of a row
        {
            const int gq = lane >> 2, tq = lane & 3;
            for (int a8 = a0 + warp * 8; a8 < a1; a8 += nwarp * 8) {
                const int arow = a8 + gq;
                const bool va = arow < a1;
                double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
                const unsigned long long ppsi = a8 < g.psi_keep ? pkeep : pstream;  // warp-uniform
                for (int ib = 0; ib < n_occ; ib += 4 * KQ_UP) {
                    double af[KQ_UP];
#pragma unroll
                    for (int u = 0; u < KQ_UP; ++u) {  // KQ_UP fragments of psi in flight
                        const int i = ib + 4 * u + tq;
                        af[u] = (va && i < n_occ) ? (g.psi_keep < 0 ? g.Psi[(size_t)i * Ng + arow]
                                                             : kq_ld_ro(&g.Psi[(size_t)i * Ng + arow], ppsi))
                                               : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < KQ_UP; ++u) {
                        const int i = ib + 4 * u + tq;
                        if (ib + 4 * u < n_occ) {  // warp-uniform
                            const double b0 = i < n_occ ? qs[i + gq * (n_occ + 4)] : 0.0;
                            dmma_kq(c0[0], c0[1], af[u], b0);
                            if (RQ > 8) {
                                const double b1 = i < n_occ ? qs[i + (8 + gq) * (n_occ + 4)] : 0.0;
                                dmma_kq(c1[0], c1[1], af[u], b1);
                            }
                        }
                    }
                }
                // this lane holds P(a8 + gq, 2 tq + {0, 1}) and P(a8 + gq, 8 + 2 tq + {0, 1})
                double part = 0.0;
                if (va) {
                    part = g.Gt[(size_t)(2 * tq) * Ng + arow] * c0[0] + g.Gt[(size_t)(2 * tq + 1) * Ng + arow] * c0[1];
                    if (RQ > 8)
                        part += g.Gt[(size_t)(8 + 2 * tq) * Ng + arow] * c1[0] +
                                g.Gt[(size_t)(9 + 2 * tq) * Ng + arow] * c1[1];
                }
                part += __shfl_xor_sync(0xffffffffu, part, 1);
                part += __shfl_xor_sync(0xffffffffu, part, 2);
                if (va && tq == 0) {
                    g.Rrows[(size_t)j * Ng + arow] = part;
                    if (!g.dn[arow]) g.n2[arow] -= part * part;
                }
            }
        }
        __syncthreads();
        // the candidates' screening norms restart from their exact values
        if (t < nc && t != wc) {
            const int a = __ldcg(&g.cand[par * KQ_CMAX + t]);
            if (a >= a0 && a < a1) {
                const double rv = g.Rrows[(size_t)j * Ng + a];
                g.n2[a] = sred[0][t] - rv * rv;
            }
        }
        __syncthreads();
        p1(j + 1);
        __threadfence();
        grid.sync();
        KQ_MARK(7);
    }
    if (b == 0 && t == 0) *g.out_nmu = N;
}

// AB = [R11 | R(0:N, :)] (N x (N + Ng), ld N) for the blocked upper-triangular solve.
__global__ void k_kq_gather(int N, int Ng, int kmax, const double* __restrict__ R11, const double* __restrict__ Rrows,
                            double* __restrict__ AB) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int col = blockIdx.y + gridDim.y * blockIdx.z;
    if (i >= N || col >= N + Ng) return;
    AB[(size_t)col * N + i] = col < N ? (i <= col ? R11[(size_t)col * kmax + i] : 0.0) : Rrows[(size_t)i * Ng + col - N];
}

// Xi(a, mu) = (R11^{-1} R(0:N, a))_mu, exactly delta(mu, pos) for the N pivots;  S = pivots.
__global__ void k_kq_xi(int N, int Ng, const double* __restrict__ T, const int* __restrict__ pos,
                        const int* __restrict__ dn, const int* __restrict__ piv, double* __restrict__ Xi,
                        int* __restrict__ S) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int mu = blockIdx.y;
    if (a >= Ng) return;
    const bool pv = dn[a] && pos[a] < N;
    Xi[(size_t)mu * Ng + a] = pv ? (pos[a] == mu ? 1.0 : 0.0) : T[(size_t)a * N + mu];
    if (a == 0) S[mu] = piv[mu];
}

bool kq_supported(int r) { return r == 8 || r == 16; }

int kq_compress(acp_context* ctx, const double* Psi, const double* Gt, int r, int kmax, double id_eps, int n_fixed,
                int n_mu_max, int* S, double* Xi) {
    const int Ng = ctx->Ng, n_occ = ctx->sys.n_occ, m = n_occ * r;
    int sms = 148;
    ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    KqArgs g;
    g.m = m;
    g.Ng = Ng;
    g.n_occ = n_occ;
    g.r = r;
    g.kmax = kmax;
    g.fixed = n_fixed;
    g.eps = id_eps;
    g.Psi = Psi;
    g.Gt = Gt;
    g.Q = ctx->wsd("kq_Q", (size_t)m * kmax);
    g.Rrows = ctx->wsd("kq_Rrows", (size_t)kmax * Ng);
    g.R11 = ctx->wsd("kq_R11", (size_t)kmax * kmax);
    g.n2 = ctx->wsd("kq_n2", Ng);
    g.pos = ctx->wsi("kq_pos", Ng);
    g.dn = ctx->wsi("kq_dn", Ng);
    g.piv = ctx->wsi("kq_piv", kmax);
    g.rdiag = ctx->wsd("kq_rdiag", kmax);
    g.slots = ctx->wsd("kq_slots", 4 * (size_t)sms);
    g.tpart = ctx->wsd("kq_tpart", 4 * (size_t)sms * KQ_CMAX);
    g.Y = ctx->wsd("kq_Y", (size_t)KQ_CMAX * m);
    g.w2 = ctx->wsd("kq_w2", kmax);
    g.cand = ctx->wsi("kq_cand", 2 * KQ_CMAX);
    g.ncand = ctx->wsi("kq_ncand", 4);
    g.out_nmu = ctx->wsi("kq_nmu", 1);
    g.overflow = ctx->wsi("kq_overflow", 1);
    {
        // share of Psi pinned in L2 across pivots (percent of the grid points; ACP_KQ_PSI_KEEP)
        static const char* e = getenv("ACP_KQ_PSI_KEEP");
        // default 0: the whole Psi pass streams evict_first, which keeps Q (the three passes per pivot)
        // L2-resident -- c4g compress 417 vs 430 ms; pinning 30 / 50 / 70 / 90 % of Psi: 427 / 430 / 432 /
        // 433 ms; Q loads evict_last: no change (run R5j).  < 0: plain loads.
        const int pct = e ? std::min(100, atoi(e)) : 0;
        g.psi_keep = pct < 0 ? -1 : (int)((long long)Ng * pct / 100);
        static const char* eq = getenv("ACP_KQ_QLAST");
        g.q_last = eq ? atoi(eq) : 0;
    }
    static const bool prof = getenv("ACP_KQ_PROF") != nullptr;
    g.prof = prof ? reinterpret_cast<long long*>(ctx->ws("kq_prof", 16 * sizeof(long long))) : nullptr;
    if (prof) ACP_CUDA(cudaMemsetAsync(g.prof, 0, 16 * sizeof(long long), ctx->stream));
    ACP_CUDA(cudaMemsetAsync(g.ncand, 0, 4 * sizeof(int), ctx->stream));
    ACP_CUDA(cudaMemsetAsync(g.overflow, 0, sizeof(int), ctx->stream));
    k_kq_init<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(Ng, n_occ, r, Psi, Gt, g.n2, g.pos, g.dn);
    launched(ctx);
    const void* fn = r == 8 ? (const void*)k_kq<8> : (const void*)k_kq<16>;
    const size_t smem = ((size_t)KQ_CMAX * (n_occ + r) + std::max(m + 4 * r, KQ_T * 4)) * sizeof(double);
    ACP_REQUIRE(smem <= 200 * 1024, "Kronecker QRCP: sketch too tall for the shared staging");
    func_attr(fn, smem);
    int occ = 0;
    ACP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, KQ_T, smem));
    ACP_REQUIRE(occ >= 1, "Kronecker QRCP: kernel does not fit");
    // resident CTAs (two per SM at <= 128 registers): the phases are latency-bound, more warps
    // keep more loads in flight (ACP_KQ_CTAS overrides for A/B)
    int G = occ * sms;
    if (const char* e = getenv("ACP_KQ_CTAS")) G = std::max(1, std::min(G, atoi(e)));
    void* args[] = {&g};
    ACP_CUDA(cudaLaunchCooperativeKernel(fn, dim3(G), dim3(KQ_T), args, smem, ctx->stream));
    launched(ctx);
    int* hp = static_cast<int*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, g.out_nmu, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaMemcpyAsync(hp + 1, g.overflow, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    const int N = hp[0];
    if (prof) {
        long long h[16];
        ACP_CUDA(cudaMemcpy(h, g.prof, sizeof(h), cudaMemcpyDeviceToHost));
        fprintf(stderr, "[kq CTA0 cycles/pivot, N=%d]", N);
        for (int q = 0; q < 8; ++q) fprintf(stderr, " %lld", N ? h[q] / N : 0);
        fprintf(stderr, "\n");
    }
    ACP_REQUIRE(hp[1] == 0, "Kronecker QRCP: more near-tied columns than the candidate buffer holds");
    ACP_REQUIRE(N >= 1, "QRCP selected no rows (zero sketch)");
    if (N > n_mu_max)
        throw Error(ACP_ERR_INVALID, "N_mu = " + std::to_string(N) + " exceeds n_mu_max = " + std::to_string(n_mu_max));
    double* AB = ctx->wsd("kq_AB", (size_t)N * (N + Ng));
    const int ncol = N + Ng, gz = cdiv(ncol, 65535);
    k_kq_gather<<<dim3(cdiv(N, 128), cdiv(ncol, gz), gz), 128, 0, ctx->stream>>>(N, Ng, kmax, g.R11, g.Rrows, AB);
    launched(ctx);
    upper_solve_blocked(ctx, AB, N, Ng);
    k_kq_xi<<<dim3(cdiv(Ng, 256), N), 256, 0, ctx->stream>>>(N, Ng, AB + (size_t)N * N, g.pos, g.dn, g.piv, Xi, S);
    launched(ctx);
    return N;
}

}  // namespace acp
