// fft.cu -- in-house fp64 FFTs and the Fourier-operator kernel (K1), 1D and 2D.
//
// The Hamiltonian apply of PAPER.md:189 (Eq. Hamil), H psi = -1/2 Delta psi + V psi,
// uses the Fourier symbol |k|^2/2 for -1/2 Delta on the periodic grid (PAPER.md:852
// "plane wave basis set"); the Yukawa operator v_hxc = K (Eq. yukawa)
// and the CG preconditioner are Fourier multipliers of the same kind.
//
// K1 computes Y = IFFT(mult . FFT(X)) + (diag - shift_j) (.) X for a batch of real
// columns.  Two real columns are packed as z = a + i b (real-even symbols keep the two
// results separable exactly), the inverse transform is conj -> forward FFT (1/N folded
// into the symbol), and the pointwise (V - shift) multiply, the activity mask and the
// per-column CG dot products are fused into the write: each column is read once and
// written once from HBM.
//   1D: one CTA per column pair, in-place Stockham FFT in shared memory (fft_engine.cuh).
//   2D (n0 x n1 grid): one thread-block CLUSTER of cs CTAs per column pair.  CTA r owns
//       rows [r n0/cs, (r+1) n0/cs): row FFTs in its shared memory, then a transpose
//       through distributed shared memory (each CTA gathers its n1/cs columns from every
//       peer), column FFTs, symbol multiply, column FFTs, transpose back, row FFTs.
//       Shared memory is indexed through P(i) = i + i/8 and the column phase uses ld = n0 + 8,
//       which makes the Stockham passes and the DSMEM transposes (nearly) bank-conflict free.  Per-column dot products are reduced over the cluster in
//       rank order (deterministic).
#include <cooperative_groups.h>

#include "fft_engine.cuh"

#include <algorithm>
#include <map>
#include <cmath>
#include <cstdlib>

namespace acp {

namespace cg = cooperative_groups;

FftPlan make_plan(int N) {
    FftPlan p;
    p.N = N;
    int n = N;
    const int order[5] = {8, 4, 2, 5, 3};
    for (int oi = 0; oi < 5; ++oi) {
        int R = order[oi];
        while (n % R == 0) {
            ACP_REQUIRE(p.npass < 24, "FFT length has too many factors");
            p.radix[p.npass++] = R;
            n /= R;
        }
    }
    ACP_REQUIRE(n == 1, "grid size must factor into 2, 3 and 5");
    int Ns = 1;
    for (int q = 0; q < p.npass; ++q) {
        p.twoff[q + 1] = p.twoff[q] + Ns * (p.radix[q] - 1);
        Ns *= p.radix[q];
    }
    return p;
}

// Geometry handed to every FFT kernel.
struct FftGeom {
    FftPlan p0, p1;   // axis 0 / axis 1 plans (1D: p0 only)
    int n0, n1;       // grid (1D: n1 = 1)
    int cs, r0, c1;   // 2D cluster size, rows and columns per CTA
    int tw0n, tw1n;   // twiddle table entries (axis 0 / axis 1)
    double dk0, dk1;  // 2 pi / L per axis
    double invN;      // 1 / N_g
    float rc1, rr0, rn1;  // float reciprocals of c1, r0, n1 for fdiv (exact for indices < 2^21)
    int np;               // 2D: column pairs per cluster
    float rper_c, rper_r; // 1 / (n0 c1), 1 / (r0 n1)
    int ldc;          // column-phase leading dimension (n0 + 8)
};

static FftGeom geom(const acp_context* ctx) {
    FftGeom g;
    g.p0 = ctx->plan;
    g.p1 = ctx->plan1;
    g.n0 = ctx->n[0];
    g.n1 = ctx->n[1];
    g.cs = ctx->cs;
    g.r0 = ctx->r0;
    g.c1 = ctx->c1;
    g.dk0 = 2.0 * M_PI / ctx->sys.cell[0];
    g.dk1 = ctx->dim == 2 ? 2.0 * M_PI / ctx->sys.cell[1] : 0.0;
    g.invN = 1.0 / (double)ctx->Ng;
    g.rc1 = ctx->c1 > 0 ? 1.0f / (float)ctx->c1 : 0.0f;
    g.rr0 = ctx->r0 > 0 ? 1.0f / (float)ctx->r0 : 0.0f;
    g.rn1 = 1.0f / (float)g.n1;
    g.np = ctx->dim == 2 ? ctx->fnp : 1;
    g.rper_c = ctx->dim == 2 ? 1.0f / (float)(g.n0 * ctx->c1) : 0.0f;
    g.rper_r = ctx->dim == 2 ? 1.0f / (float)(ctx->r0 * g.n1) : 0.0f;
    g.tw0n = g.p0.twoff[g.p0.npass];
    g.tw1n = ctx->dim == 2 ? g.p1.twoff[g.p1.npass] : 0;
    g.ldc = g.n0 + 8;  // with the P() pad: conflict-free column passes and transposes (enumerated)
    return g;
}

// I/O modes of the FFT kernels.
enum { IO_OP = 0, IO_HERM = 1, IO_SPEC = 2 };

struct IoArgs {
    FopArgs f;                  // IO_OP
    const double2* spec = nullptr;  // IO_HERM: n spectra (N_g complex each)
    double* out = nullptr;      // IO_HERM: n real columns
    double scale = 1.0;         // IO_HERM
    const double* x = nullptr;  // IO_SPEC: one real column
    double2* sout = nullptr;    // IO_SPEC: its spectrum
    int n = 0;                  // number of columns (IO_OP: f.n)
};

// In-kernel symbol of bin (i0, i1) (already divided by N, like the tables).
__device__ __forceinline__ double sym_value(const FftGeom& G, int sym, double tau, int i0, int i1) {
    const int m0 = i0 < (G.n0 + 1) / 2 ? i0 : i0 - G.n0;
    const int m1 = i1 < (G.n1 + 1) / 2 ? i1 : i1 - G.n1;
    const double ka = m0 * G.dk0, kb = m1 * G.dk1;
    const double h = 0.5 * (ka * ka + kb * kb);
    if (sym == MULT_KINETIC) return h * G.invN;
    // MULT_PRECOND: 1/(h + tau) by the hardware reciprocal estimate refined by two Newton steps
    const double d = h + tau;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = r * (2.0 - d * r);
    r = r * (2.0 - d * r);
    return r * G.invN;
}

// ============================================================================ 1D

// One CTA per column pair.  Shared memory: the padded FFT buffer, the twiddle table and (IO_OP)
// the multiplier, which is copied with cp.async at kernel start and consumed after the first FFT.
// Each thread keeps its input values (i = tid + q T) in registers for the epilogue and
// prefetches the potential before the second FFT, so no global load sits on the critical path
// after the initial one.
// NCT != 0: the FFT length is the compile-time constant NCT (fft_ct), else the runtime plan.
template <int EPT, bool KEEP, int IO, int NCT = 0, int NKT = 1024, int NKB = 1>
__global__ void __launch_bounds__(KEEP ? 160 : NKT, KEEP ? 4 : NKB) k_fft1d(FftGeom G, const double2* __restrict__ twg,
                                                             IoArgs io) {
    extern __shared__ __align__(16) double2 sm1[];
    __shared__ double red[132];
    const int N = G.n0;
    const int T = blockDim.x, tid = threadIdx.x;
    double2* buf = sm1;
    double* smult = reinterpret_cast<double*>(sm1 + padded(N));
    const int c0 = 2 * blockIdx.x, c1 = c0 + 1;
    const int ncol = IO == IO_OP ? io.f.n : io.n;
    const bool has1 = c1 < ncol;
    pdl_wait();
    pdl_trigger();
    bool act0 = true, act1 = has1;
    if (IO == IO_OP && io.f.active) {
        act0 = io.f.active[c0] != 0;
        act1 = has1 && io.f.active[c1] != 0;
    }
    if (!act0 && !act1) return;
#define K1_TP(q) \
    if (IO == IO_OP && io.f.tprof && blockIdx.x == 0 && threadIdx.x == 0) io.f.tprof[q] = clock64();
    K1_TP(0)
    const bool do_fft = IO != IO_OP || io.f.mult != nullptr || io.f.sym >= 0;
    if (IO == IO_OP && io.f.mult && io.f.sym < 0) {
        if ((N & 1) == 0) {
            for (int c = tid; c < N / 2; c += T) cp_async16_fe(smult + 2 * c, io.f.mult + 2 * c);
        } else {
            for (int i = tid; i < N; i += T) smult[i] = io.f.mult[i];
        }
    }
    // twiddles are read through L1 (read-only path): staging the 20 KB table in shared memory
    // cost a CTA per SM (measured 10 % slower on configs[1] / [2], profiles/r2i)
    const double2* tw = twg;
    constexpr int NK = KEEP ? EPT : 1;  // register-resident inputs (KEEP) or re-read in the epilogue
    double u0[NK], u1[NK];
    const double* x0 = io.f.X + (size_t)c0 * N;
    const double* x1 = io.f.X + (size_t)c1 * N;
    if (IO == IO_OP && KEEP) {
#pragma unroll
        for (int q = 0; q < NK; ++q) {
            const int i = tid + q * T;
            u0[q] = i < N ? x0[i] : 0.0;
            u1[q] = (i < N && has1) ? x1[i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < NK; ++q) {
            const int i = tid + q * T;
            if (i < N) buf[P(i)] = make_double2(u0[q], u1[q]);
        }
    } else if (IO == IO_OP) {
        for (int i = tid; i < N; i += T) buf[P(i)] = make_double2(x0[i], has1 ? x1[i] : 0.0);
    } else if (IO == IO_HERM) {
        const double2* s0 = io.spec + (size_t)c0 * N;
        const double2* s1 = io.spec + (size_t)c1 * N;
        for (int i = tid; i < N; i += T) {
            const double2 p = s0[i];
            const double2 q = has1 ? s1[i] : make_double2(0.0, 0.0);
            buf[P(i)] = make_double2(p.x - q.y, -(p.y + q.x));  // conj(P + i Q)
        }
    } else {
        for (int i = tid; i < N; i += T) buf[P(i)] = make_double2(io.x[i], 0.0);
    }
    cp_async_wait_all_fe();  // twiddles and the multiplier
    __syncthreads();
    K1_TP(1)
    if (do_fft) {
        if constexpr (NCT != 0) fft_ct<NCT, EPT>(buf, tw);
        else fft_inplace<EPT>(buf, N, 1, G.p0, tw);
    }
    K1_TP(2)
    if (IO == IO_HERM) {
        for (int i = tid; i < N; i += T) {
            const double2 v = buf[P(i)];
            io.out[(size_t)c0 * N + i] = v.x * io.scale;
            if (has1) io.out[(size_t)c1 * N + i] = -v.y * io.scale;
        }
        return;
    }
    if (IO == IO_SPEC) {
        for (int i = tid; i < N; i += T) io.sout[i] = buf[P(i)];
        return;
    }
    const FopArgs& a = io.f;
    double dv[NK];
    if (KEEP) {
#pragma unroll
        for (int q = 0; q < NK; ++q) {
            const int i = tid + q * T;
            dv[q] = (a.diag && i < N) ? __ldg(&a.diag[i]) : 0.0;  // consumed after the second FFT
        }
    }
    if (do_fft) {
        // conj(mult * F) then forward FFT == N * conj(IFFT(mult * F)) (1/N folded into mult)
        for (int i = tid; i < N; i += T) {
            const double m = a.sym >= 0 ? sym_value(G, a.sym, a.tau, i, 0) : smult[i];
            const double2 v = buf[P(i)];
            buf[P(i)] = make_double2(m * v.x, -m * v.y);
        }
        __syncthreads();
        K1_TP(3)
        if constexpr (NCT != 0) fft_ct<NCT, EPT>(buf, tw);
        else fft_inplace<EPT>(buf, N, 1, G.p0, tw);
    }
    K1_TP(4)
    const double s0 = a.shift ? a.shift[c0] : 0.0;
    const double s1 = (a.shift && has1) ? a.shift[c1] : 0.0;
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    double* y0 = a.Y + (size_t)c0 * N;
    double* y1 = a.Y + (size_t)c1 * N;
    const int nq = KEEP ? NK : (N + T - 1) / T;
#pragma unroll(KEEP ? NK : 1)
    for (int q = 0; q < nq; ++q) {
        const int i = tid + q * T;
        if (i < N) {
            const double xa = KEEP ? u0[KEEP ? q : 0] : x0[i];
            const double xb = KEEP ? u1[KEEP ? q : 0] : (has1 ? x1[i] : 0.0);
            const double dg = KEEP ? dv[KEEP ? q : 0] : (a.diag ? a.diag[i] : 0.0);
            double v0 = 0.0, v1 = 0.0;
            if (do_fft) {
                const double2 v = buf[P(i)];
                v0 = v.x;
                v1 = -v.y;
            }
            v0 += (dg - s0) * xa;
            v1 += (dg - s1) * xb;
            if (act0) y0[i] = v0;
            if (act1) y1[i] = v1;
            d[0] += xa * v0;
            d[1] += xa * xa;
            d[2] += xb * v1;
            d[3] += xb * xb;
        }
    }
    K1_TP(5)
    if (a.dots) {
        block_sum4(d, red);
        if (tid == 0) {
            if (act0) {
                a.dots[2 * c0] = d[0];
                a.dots[2 * c0 + 1] = d[1];
            }
            if (act1) {
                a.dots[2 * c1] = d[2];
                a.dots[2 * c1 + 1] = d[3];
            }
        }
    }
    K1_TP(6)
}

// ============================================================================ 2D
// A cluster processes np column pairs (np <= 4) at once: the slices of the np pairs are stored
// back to back, so the FFT passes see np*r0 rows / np*c1 columns as ONE batch and each cluster
// barrier and DSMEM round trip is amortised over np pairs.
// Row phase: buf[(p r0 + il) n1 + k1];  column phase: buf[(p c1 + c) ldc + k0]  (P-padded).
// Transposes: one cluster barrier before the remote reads (peers finished writing), one after
// (peers may overwrite their buffer).
constexpr int NPMAX = 4;

template <int EPT>
__device__ __forceinline__ void rows_to_cols(cg::cluster_group& cl, double2* buf, const FftGeom& G, int rank) {
    double2 v[EPT];
    const int per = G.n0 * G.c1;
    const int E = G.np * per;
    cl.sync();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = threadIdx.x + q * blockDim.x;
        if (e < E) {
            const int p = fdiv(e, G.rper_c), r = e - p * per;
            const int i = fdiv(r, G.rc1), c = r - i * G.c1;
            const int src = fdiv(i, G.rr0), il = i - src * G.r0;
            const double2* rb = cl.map_shared_rank(buf, src);
            v[q] = rb[P((p * G.r0 + il) * G.n1 + rank * G.c1 + c)];
        }
    }
    cl.sync();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = threadIdx.x + q * blockDim.x;
        if (e < E) {
            const int p = fdiv(e, G.rper_c), r = e - p * per;
            const int i = fdiv(r, G.rc1), c = r - i * G.c1;
            buf[P((p * G.c1 + c) * G.ldc + i)] = v[q];
        }
    }
    __syncthreads();
}

template <int EPT>
__device__ __forceinline__ void cols_to_rows(cg::cluster_group& cl, double2* buf, const FftGeom& G, int rank) {
    double2 v[EPT];
    const int per = G.r0 * G.n1;
    const int E = G.np * per;
    cl.sync();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = threadIdx.x + q * blockDim.x;
        if (e < E) {
            const int p = fdiv(e, G.rper_r), r = e - p * per;
            const int il = fdiv(r, G.rn1), k1 = r - il * G.n1;
            const int src = fdiv(k1, G.rc1), c = k1 - src * G.c1;
            const double2* rb = cl.map_shared_rank(buf, src);
            v[q] = rb[P((p * G.c1 + c) * G.ldc + rank * G.r0 + il)];
        }
    }
    cl.sync();
#pragma unroll
    for (int q = 0; q < EPT; ++q) {
        const int e = threadIdx.x + q * blockDim.x;
        if (e < E) buf[P(e)] = v[q];
    }
    __syncthreads();
}

// np column pairs (or spectrum pairs / single columns when np = 1) per cluster; grid (cs, groups).
template <int EPT, int IO>
__global__ void __launch_bounds__(1024) k_fft2d(FftGeom G, const double2* __restrict__ tw0g,
                                               const double2* __restrict__ tw1g, IoArgs io, int grp0) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double2 sm2[];
    __shared__ double red[132];
    __shared__ double part[4 * NPMAX];
    const int rank = (int)cl.block_rank();
    const int N = G.n0 * G.n1;
    const int np = G.np;
    const int bufn = padded(np * (G.c1 * G.ldc > G.r0 * G.n1 ? G.c1 * G.ldc : G.r0 * G.n1));
    double2* buf = sm2;
    const int pbase = (grp0 + blockIdx.y) * np;  // first pair of this cluster
    const int ncol = IO == IO_OP ? io.f.n : io.n;
    pdl_wait();
    pdl_trigger();
    bool any = false;
    for (int p = 0; p < np; ++p) {
        const int c0 = 2 * (pbase + p), c1 = c0 + 1;
        if (c0 < ncol && (IO != IO_OP || !io.f.active || io.f.active[c0])) any = true;
        if (c1 < ncol && (IO != IO_OP || !io.f.active || io.f.active[c1])) any = true;
    }
    if (!any) return;  // uniform over the cluster
#define K2D_TP(q) \
    if (IO == IO_OP && io.f.tprof && blockIdx.y == 0 && rank == 0 && threadIdx.x == 0) io.f.tprof[q] = clock64();
    K2D_TP(0)
    const double2* tw0 = load_twiddles(sm2 + bufn, tw0g, G.p0);
    const double2* tw1 = load_twiddles(sm2 + bufn + G.tw0n, tw1g, G.p1);
    const int E1 = G.r0 * G.n1;           // elements of one pair owned in the row phase
    const size_t rowbase = (size_t)rank * G.r0 * G.n1;
    for (int p = 0; p < np; ++p) {
        const int c0 = 2 * (pbase + p), c1 = c0 + 1;
        const bool h0 = c0 < ncol, h1 = c1 < ncol;
        double2* bp = buf;
        const int off = p * E1;
        if (IO == IO_OP) {
            const double* x0 = io.f.X + (size_t)c0 * N + rowbase;
            const double* x1 = io.f.X + (size_t)c1 * N + rowbase;
            for (int e = threadIdx.x; e < E1; e += blockDim.x)
                bp[P(off + e)] = make_double2(h0 ? x0[e] : 0.0, h1 ? x1[e] : 0.0);
        } else if (IO == IO_HERM) {
            const double2* s0 = io.spec + (size_t)c0 * N + rowbase;
            const double2* s1 = io.spec + (size_t)c1 * N + rowbase;
            for (int e = threadIdx.x; e < E1; e += blockDim.x) {
                const double2 a = h0 ? s0[e] : make_double2(0.0, 0.0);
                const double2 b = h1 ? s1[e] : make_double2(0.0, 0.0);
                bp[P(off + e)] = make_double2(a.x - b.y, -(a.y + b.x));
            }
        } else {
            for (int e = threadIdx.x; e < E1; e += blockDim.x) bp[P(off + e)] = make_double2(io.x[rowbase + e], 0.0);
        }
    }
    cp_async_wait_all_fe();  // twiddles
    __syncthreads();
    K2D_TP(1)
    const bool do_fft = IO != IO_OP || io.f.mult != nullptr || io.f.sym >= 0;
    if (do_fft) {
        fft_inplace<EPT>(buf, G.n1, np * G.r0, G.p1, tw1);       // rows (length n1)
        K2D_TP(2)
        rows_to_cols<EPT>(cl, buf, G, rank);
        K2D_TP(3)
        fft_inplace<EPT>(buf, G.ldc, np * G.c1, G.p0, tw0);      // columns (length n0)
        K2D_TP(4)
    }
    const int Ec1 = G.n0 * G.c1;  // elements of one pair owned in the column phase
    if (IO == IO_HERM || IO == IO_SPEC) {
        // write from the column phase: bin / point (k0, k1 = rank c1 + c) -> k0 n1 + k1  (np = 1)
        const int c0 = 2 * pbase, c1 = c0 + 1;
        for (int e = threadIdx.x; e < Ec1; e += blockDim.x) {
            const int k0 = fdiv(e, G.rc1), c = e - k0 * G.c1;
            const double2 v = buf[P(c * G.ldc + k0)];
            const size_t o = (size_t)k0 * G.n1 + rank * G.c1 + c;
            if (IO == IO_SPEC) {
                io.sout[o] = v;
            } else {
                if (c0 < ncol) io.out[(size_t)c0 * N + o] = v.x * io.scale;
                if (c1 < ncol) io.out[(size_t)c1 * N + o] = -v.y * io.scale;
            }
        }
        return;  // the last remote read (rows_to_cols) is behind a cluster barrier
    }
    const FopArgs& a = io.f;
    if (do_fft) {
        for (int e = threadIdx.x; e < np * Ec1; e += blockDim.x) {
            const int p = fdiv(e, G.rper_c), r = e - p * Ec1;
            const int k0 = fdiv(r, G.rc1), c = r - k0 * G.c1;
            const double m = a.sym >= 0 ? sym_value(G, a.sym, a.tau, k0, rank * G.c1 + c)
                                        : __ldg(&a.mult[(size_t)k0 * G.n1 + rank * G.c1 + c]);
            const int o = P((p * G.c1 + c) * G.ldc + k0);
            const double2 v = buf[o];
            buf[o] = make_double2(m * v.x, -m * v.y);
        }
        __syncthreads();
        K2D_TP(5)
        fft_inplace<EPT>(buf, G.ldc, np * G.c1, G.p0, tw0);      // columns
        K2D_TP(6)
        cols_to_rows<EPT>(cl, buf, G, rank);
        K2D_TP(7)
        fft_inplace<EPT>(buf, G.n1, np * G.r0, G.p1, tw1);       // rows
        K2D_TP(8)
    }
    const double* dg = a.diag ? a.diag + rowbase : nullptr;
    for (int p = 0; p < np; ++p) {
        const int c0 = 2 * (pbase + p), c1 = c0 + 1;
        const bool h0 = c0 < ncol, h1 = c1 < ncol;
        const bool act0 = h0 && (!a.active || a.active[c0]);
        const bool act1 = h1 && (!a.active || a.active[c1]);
        const double s0 = (a.shift && h0) ? a.shift[c0] : 0.0;
        const double s1 = (a.shift && h1) ? a.shift[c1] : 0.0;
        const double* x0 = a.X + (size_t)c0 * N + rowbase;
        const double* x1 = a.X + (size_t)c1 * N + rowbase;
        double* y0 = a.Y + (size_t)c0 * N + rowbase;
        double* y1 = a.Y + (size_t)c1 * N + rowbase;
        double d[4] = {0.0, 0.0, 0.0, 0.0};
        const int off = p * E1;
        for (int e = threadIdx.x; e < E1; e += blockDim.x) {
            const double u0 = h0 ? x0[e] : 0.0;
            const double u1 = h1 ? x1[e] : 0.0;
            double v0 = 0.0, v1 = 0.0;
            if (do_fft) {
                const double2 v = buf[P(off + e)];
                v0 = v.x;
                v1 = -v.y;
            }
            if (dg) {
                const double w = dg[e];
                v0 += (w - s0) * u0;
                v1 += (w - s1) * u1;
            } else if (a.shift) {
                v0 -= s0 * u0;
                v1 -= s1 * u1;
            }
            if (act0) y0[e] = v0;
            if (act1) y1[e] = v1;
            d[0] += u0 * v0;
            d[1] += u0 * u0;
            d[2] += u1 * v1;
            d[3] += u1 * u1;
        }
        if (a.dots) {
            block_sum4(d, red);
            if (threadIdx.x < 4) part[4 * p + threadIdx.x] = d[threadIdx.x];
        }
    }
    K2D_TP(9)
    if (a.dots) {
        cl.sync();
        if (rank == 0 && threadIdx.x < 4 * np) {
            const int p = threadIdx.x >> 2, qd = threadIdx.x & 3;
            double sum = 0.0;
            for (int q = 0; q < G.cs; ++q) sum += cl.map_shared_rank(part, q)[threadIdx.x];  // rank order
            const int col = 2 * (pbase + p) + (qd >> 1);
            if (col < ncol && (!a.active || a.active[col])) a.dots[2 * col + (qd & 1)] = sum;
        }
        cl.sync();
    }
}

// ============================================================================ launchers
// shared-memory / cluster-size attributes once per (device, kernel instance) and size (a host call
// per launch would make the un-graphed launches host-bound)
static void set_smem_attr(const void* kern, size_t smem, bool cluster16) { func_attr(kern, smem, cluster16); }

template <int IO>
static void launch_fft(acp_context* ctx, const IoArgs& io, int ncols) {
    if (ncols <= 0) return;
    const FftGeom G = geom(ctx);
    const int npair = (ncols + 1) / 2;
    const int T = ctx->fthreads;
    size_t smem = ctx->fsmem;
    if (ctx->dim == 1) {
        // the multiplier-table region is needed only when the symbol comes from a table
        const bool table = IO == IO_OP && io.f.mult != nullptr && io.f.sym < 0;
        if (!table) smem = (size_t)padded(G.n0) * sizeof(double2);
        // KEEP (register-resident inputs, <= 160 threads, 4 CTAs/SM) for N <= 1280 (without: configs[1]
        // 11.75 vs 11.58 ms/step)
        auto kern = T > 160 ? (ctx->fept <= 8 ? k_fft1d<8, false, IO> : k_fft1d<16, false, IO>)
                  : ctx->fept <= 2 ? k_fft1d<2, true, IO> : ctx->fept <= 4 ? k_fft1d<4, true, IO>
                  : k_fft1d<8, true, IO>;
        // compiled-length kernels for the configs' grids (hot path only; ACP_FFT_GENERIC=1 off)
        if (IO == IO_OP && ctx->fct) {
            if (G.n0 == 1280 && T <= 160 && ctx->fept == 8) kern = k_fft1d<8, true, IO, 1280>;
            else if (G.n0 == 960 && T <= 160 && ctx->fept == 8) kern = k_fft1d<8, true, IO, 960>;
            else if (G.n0 == 256 && T <= 160 && ctx->fept == 4) kern = k_fft1d<4, true, IO, 256>;
            else if (G.n0 == 5120 && T > 160 && ctx->fept == 8)
                // 2 CTAs/SM (<= 48 registers): K1 400 vs 474 us, configs[2] 241 vs 251 ms/step
                kern = T == 640 ? k_fft1d<8, false, IO, 5120, 640, 2> : k_fft1d<8, false, IO, 5120>;
        }
        set_smem_attr((const void*)kern, ctx->fsmem, false);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(npair, 1, 1);
        cfg.blockDim = dim3(T, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = ctx->pdl ? 1 : 0;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, G, (const double2*)ctx->d_tw, io));
        launched(ctx);
        return;
    }
    FftGeom Gl = G;
    if (IO != IO_OP) Gl.np = 1;  // setup transforms: one pair per cluster
    const int ept = IO == IO_OP ? ctx->fept : ctx->fept1;
    const int Tl = IO == IO_OP ? T : ctx->fthreads1;
    const size_t smeml = IO == IO_OP ? smem : ctx->fsmem1;
    auto kern = ept <= 2 ? k_fft2d<2, IO> : ept <= 4 ? k_fft2d<4, IO> : ept <= 8 ? k_fft2d<8, IO> : k_fft2d<16, IO>;
    set_smem_attr((const void*)kern, smeml, true);
    const int ngrp = (npair + Gl.np - 1) / Gl.np;
    for (int g0 = 0; g0 < ngrp; g0 += 32768) {
        const int ng = ngrp - g0 < 32768 ? ngrp - g0 : 32768;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctx->cs, ng, 1);
        cfg.blockDim = dim3(Tl, 1, 1);
        cfg.dynamicSmemBytes = smeml;
        cfg.stream = ctx->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = ctx->cs;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = ctx->pdl ? 2 : 1;
        ACP_CUDA(cudaLaunchKernelEx(&cfg, kern, Gl, (const double2*)ctx->d_tw, (const double2*)ctx->d_tw1, io, g0));
        launched(ctx);
    }
}

// ============================================================================ 2D, three passes
// K1 for 2D grids as three grid-wide passes through an HBM/L2 intermediate Z (one complex field
// per column pair, layout [i0][k1]) instead of one thread-block cluster per pair: the cluster
// kernel spends its time in cluster barriers and index arithmetic (ncu, profiles/r1zu), while
// each pass here is a plain batched 1D FFT with coalesced 8-column / 8-row tiles.
//   A  rows:    Z[i0][.] = FFT_row(x0 + i x1)               (RB = 8 rows of one pair per CTA)
//   B  columns: Z[.][k1] = FFT_col(conj(m (.) FFT_col(Z)))  (CB = 8 columns of one pair per CTA)
//   C  rows:    y = conj(FFT_row(Z)) + (V - shift) x, per-CTA partial dots; k_f2_dots sums the
//               partials of a column in row-block order (fixed order, deterministic).
// Same transform and inverse-by-conjugation as k_fft2d; different rounding order.
constexpr int F2_RB = 8, F2_CB = 8;  // 8 x n values per CTA: <= 256 threads, 3 CTAs/SM
// Z is stored in 8 x 8 tiles (tile (i0/8, k1/8) at ((i0/8) n1/8 + k1/8) * 64, row-major inside),
// so a row block (passes A, C) is one contiguous range and a column block (pass B) is n0/8
// contiguous 1 KB tiles instead of n0 strided 128-byte segments.
static_assert(F2_RB == 8 && F2_CB == 8, "the tiled intermediate assumes 8-row / 8-column blocks");

__device__ __forceinline__ bool f2_pair_active(const FopArgs& a, int c0) {
    const bool h1 = c0 + 1 < a.n;
    return !a.active || a.active[c0] || (h1 && a.active[c0 + 1]);
}

// NCT != 0: square grid n0 = n1 = NCT with compile-time FFT indexing (fft_ct).
template <int EPT, int NCT = 0, int TB = 256, int MB = 3>
__global__ void __launch_bounds__(TB, MB) k_f2_rows_fwd(FftGeom G, const double2* __restrict__ twg, FopArgs a,
                                                     double2* __restrict__ Z, int pair0) {
    extern __shared__ __align__(16) double2 f2s[];
    const int pr = pair0 + blockIdx.y, c0 = 2 * pr;
    if (!f2_pair_active(a, c0)) return;
    const int n1 = G.n1, N = G.n0 * n1, E = F2_RB * n1;
    double2* buf = f2s;
    const double2* tw = load_twiddles(f2s + padded(E), twg, G.p1);
    const size_t rb = (size_t)blockIdx.x * E;
    const bool h1 = c0 + 1 < a.n;
    const double* x0 = a.X + (size_t)c0 * N + rb;
    const double* x1 = a.X + (size_t)(c0 + 1) * N + rb;
    for (int e = threadIdx.x; e < E; e += blockDim.x) buf[P(e)] = make_double2(x0[e], h1 ? x1[e] : 0.0);
    cp_async_wait_all_fe();
    __syncthreads();
    if constexpr (NCT != 0) fft_ct<NCT, EPT, F2_RB, NCT>(buf, tw);
    else fft_inplace<EPT>(buf, n1, F2_RB, G.p1, tw);
    double2* z = Z + (size_t)blockIdx.y * N + rb;  // this row block: E contiguous values (8 x 8 tiles)
    for (int o = threadIdx.x; o < E; o += blockDim.x) {
        const int r = (o >> 3) & 7, k1 = ((o >> 6) << 3) | (o & 7);
        z[o] = buf[P(r * n1 + k1)];
    }
}

template <int EPT, int NCT = 0, int TB = 256, int MB = 3>
__global__ void __launch_bounds__(TB, MB) k_f2_cols(FftGeom G, const double2* __restrict__ twg, FopArgs a,
                                                 double2* __restrict__ Z, int pair0) {
    extern __shared__ __align__(16) double2 f2s[];
    const int pr = pair0 + blockIdx.y, c0 = 2 * pr;
    if (!f2_pair_active(a, c0)) return;
    const int n0 = G.n0, n1 = G.n1, ld = G.ldc, E = F2_CB * n0;
    double2* buf = f2s;
    const double2* tw = load_twiddles(f2s + padded(F2_CB * ld), twg, G.p0);
    const int k1b = blockIdx.x * F2_CB;
    // column block k1b / 8: tiles (ib, k1b / 8) for ib = 0 .. n0/8 - 1, 64 contiguous values each
    double2* z = Z + (size_t)blockIdx.y * n0 * n1 + (size_t)blockIdx.x * 64;
    const int tstride = (n1 / 8) * 64;
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int ib = e >> 6, w = e & 63;
        const int i0 = (ib << 3) | (w >> 3), c = w & 7;
        buf[P(c * ld + i0)] = z[(size_t)ib * tstride + w];
    }
    cp_async_wait_all_fe();
    __syncthreads();
    if constexpr (NCT != 0) fft_ct<NCT, EPT, F2_CB, NCT + 8>(buf, tw);
    else fft_inplace<EPT>(buf, ld, F2_CB, G.p0, tw);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int c = e / n0, k0 = e - c * n0;
        const int k1 = k1b + c;
        const double m = a.sym >= 0 ? sym_value(G, a.sym, a.tau, k0, k1) : __ldg(&a.mult[(size_t)k0 * n1 + k1]);
        const int o = P(c * ld + k0);
        const double2 v = buf[o];
        buf[o] = make_double2(m * v.x, -m * v.y);
    }
    __syncthreads();
    if constexpr (NCT != 0) fft_ct<NCT, EPT, F2_CB, NCT + 8>(buf, tw);
    else fft_inplace<EPT>(buf, ld, F2_CB, G.p0, tw);
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const int ib = e >> 6, w = e & 63;
        const int i0 = (ib << 3) | (w >> 3), c = w & 7;
        z[(size_t)ib * tstride + w] = buf[P(c * ld + i0)];
    }
}

template <int EPT, int NCT = 0, int TB = 256, int MB = 3>
__global__ void __launch_bounds__(TB, MB) k_f2_rows_inv(FftGeom G, const double2* __restrict__ twg, FopArgs a,
                                                     const double2* __restrict__ Z, int pair0,
                                                     double* __restrict__ part) {
    extern __shared__ __align__(16) double2 f2s[];
    __shared__ double red[132];
    const int pr = pair0 + blockIdx.y, c0 = 2 * pr, c1 = c0 + 1;
    if (!f2_pair_active(a, c0)) return;
    const int n1 = G.n1, N = G.n0 * n1, E = F2_RB * n1;
    double2* buf = f2s;
    const double2* tw = load_twiddles(f2s + padded(E), twg, G.p1);
    const size_t rb = (size_t)blockIdx.x * E;
    const double2* z = Z + (size_t)blockIdx.y * N + rb;  // this row block (8 x 8 tiles)
    for (int o = threadIdx.x; o < E; o += blockDim.x) {
        const int r = (o >> 3) & 7, k1 = ((o >> 6) << 3) | (o & 7);
        buf[P(r * n1 + k1)] = z[o];
    }
    cp_async_wait_all_fe();
    __syncthreads();
    if constexpr (NCT != 0) fft_ct<NCT, EPT, F2_RB, NCT>(buf, tw);
    else fft_inplace<EPT>(buf, n1, F2_RB, G.p1, tw);
    const bool h1 = c1 < a.n;
    const bool act0 = !a.active || a.active[c0];
    const bool act1 = h1 && (!a.active || a.active[c1]);
    const double s0 = a.shift ? a.shift[c0] : 0.0;
    const double s1 = (a.shift && h1) ? a.shift[c1] : 0.0;
    const double* x0 = a.X + (size_t)c0 * N + rb;
    const double* x1 = a.X + (size_t)c1 * N + rb;
    double* y0 = a.Y + (size_t)c0 * N + rb;
    double* y1 = a.Y + (size_t)c1 * N + rb;
    const double* dg = a.diag ? a.diag + rb : nullptr;
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    for (int e = threadIdx.x; e < E; e += blockDim.x) {
        const double u0 = x0[e];
        const double u1 = h1 ? x1[e] : 0.0;
        const double2 v = buf[P(e)];
        double v0 = v.x, v1 = -v.y;
        if (dg) {
            const double w = dg[e];
            v0 += (w - s0) * u0;
            v1 += (w - s1) * u1;
        } else if (a.shift) {
            v0 -= s0 * u0;
            v1 -= s1 * u1;
        }
        if (act0) y0[e] = v0;
        if (act1) y1[e] = v1;
        d[0] += u0 * v0;
        d[1] += u0 * u0;
        d[2] += u1 * v1;
        d[3] += u1 * u1;
    }
    if (a.dots) {
        block_sum4(d, red);
        if (threadIdx.x < 4) part[((size_t)pr * gridDim.x + blockIdx.x) * 4 + threadIdx.x] = d[threadIdx.x];
    }
}

// dots[2c + q] = sum over row blocks (in order) of the pair's partials, active columns only.
__global__ void k_f2_dots(int n, int nrb, const double* __restrict__ part, const int* __restrict__ active,
                          double* __restrict__ dots) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (column, q)
    if (i >= 2 * n) return;
    const int col = i >> 1, q = i & 1;
    if (active && !active[col]) return;
    const int pr = col >> 1, w = 2 * (col & 1) + q;
    double s = 0.0;
    for (int b = 0; b < nrb; ++b) s += part[((size_t)pr * nrb + b) * 4 + w];
    dots[i] = s;
}

// Workspace of the three-pass 2D operator for n columns, allocated ahead of a stream capture
// (allocation is not permitted while capturing).
static std::string f2_name(const char* base, int alt) { return alt ? base + std::to_string(alt) : std::string(base); }

// The fused operator (fft2c.cu) is the default where it measured faster: 256^2 (configs[4] grid,
// K1 3.01 vs 4.07 ms per 4096 columns) and the small test grids; on 192^2 (configs[3]) it is on par
// with the three passes (4.57 vs 4.49 ms per 7680 columns, profiles/R2i_k1.txt), which stay.
// ACP_F2C=0 / 1 forces either path.
static bool use_f2c(const acp_context* ctx) {
    if (ctx->dim != 2 || !ctx->d_twf2c) return false;
    static const char* e = getenv("ACP_F2C");
    if (e) return atoi(e) != 0;
    return ctx->n[0] != 192;
}

void fourier_reserve(acp_context* ctx, int n, int alt) {
    if (ctx->dim != 2 || n <= 0) return;
    const int npair = (n + 1) / 2;
    if (use_f2c(ctx)) {
        ctx->ws(f2_name("f2c_S", alt), f2c_scratch_bytes(ctx, n));
        ctx->wsi(f2_name("f2c_q", alt), f2c_queue_ints(n));
        ctx->wsd(f2_name("f2_part", alt), (size_t)npair * f2c_items_per_phase(ctx->n[0]) * 4);
        return;
    }
    ctx->ws(f2_name("f2_Z", alt), (size_t)npair * ctx->n[0] * ctx->n[1] * sizeof(double2));
    ctx->wsd(f2_name("f2_part", alt), (size_t)npair * (ctx->n[0] / F2_RB) * 4);
}

static bool launch_fft2d_passes(acp_context* ctx, const FopArgs& a) {
    const FftGeom G = geom(ctx);
    const int n0 = G.n0, n1 = G.n1;
    if (getenv("ACP_FFT2D_CLUSTER") || n0 % F2_RB || n1 % F2_CB) return false;
    if (a.mult == nullptr && a.sym < 0) return false;  // no transform: the cluster kernel's epilogue only
    const int npair = (a.n + 1) / 2;
    const int Tr = std::min(256, std::max(64, (F2_RB * n1 / 8 + 31) / 32 * 32));
    const int Tc = std::min(256, std::max(64, (F2_CB * n0 / 8 + 31) / 32 * 32));
    const int er = (F2_RB * n1 + Tr - 1) / Tr, ec = (F2_CB * n0 + Tc - 1) / Tc;
    if (er > 16 || ec > 16) return false;
    const size_t sr = (size_t)(padded(F2_RB * n1) + G.tw1n) * sizeof(double2);
    const size_t sc = (size_t)(padded(F2_CB * G.ldc) + G.tw0n) * sizeof(double2);
    if (sr > 200 * 1024 || sc > 200 * 1024) return false;
    const int nrb = n0 / F2_RB, ncb = n1 / F2_CB;
    // each concurrent PCG group (its own stream, ctx->f2_alt) has its own intermediate
    double2* Z = static_cast<double2*>(ctx->ws(f2_name("f2_Z", ctx->f2_alt), (size_t)npair * n0 * n1 * sizeof(double2)));
    double* part = a.dots ? ctx->wsd(f2_name("f2_part", ctx->f2_alt), (size_t)npair * nrb * 4) : nullptr;
    auto ra = er <= 8 ? k_f2_rows_fwd<8> : k_f2_rows_fwd<16>;
    auto cb = ec <= 8 ? k_f2_cols<8> : k_f2_cols<16>;
    auto rc = er <= 8 ? k_f2_rows_inv<8> : k_f2_rows_inv<16>;
    // compiled-length kernels for the square configs grids (plans checked in fft_init)
    if (ctx->fct && n0 == n1 && er <= 8 && ec <= 8) {
        if (n0 == 192) {
            // 192 threads per CTA bounded to 6 CTAs/SM (<= 56 registers, no spill): configs[3]
            // 762 / 787 / 825 ms/step at 6 / 5 / 3 CTAs/SM
            ra = k_f2_rows_fwd<8, 192, 192, 6>;
            cb = k_f2_cols<8, 192, 192, 6>;
            rc = k_f2_rows_inv<8, 192, 192, 6>;
        } else if (n0 == 256) {
            // 256 threads bounded to 5 CTAs/SM (<= 48 registers, small spills): K1 4.06 / 4.51 / 5.31
            // ms at 4096 columns for 5 / 4 / 3 CTAs/SM
            ra = k_f2_rows_fwd<8, 256, 256, 5>;
            cb = k_f2_cols<8, 256, 256, 5>;
            rc = k_f2_rows_inv<8, 256, 256, 5>;
        }
    }
    set_smem_attr((const void*)ra, sr, false);
    set_smem_attr((const void*)cb, sc, false);
    set_smem_attr((const void*)rc, sr, false);
    const double2* tw0 = (const double2*)ctx->d_tw;
    const double2* tw1 = (const double2*)ctx->d_tw1;
    const int chunk = 65535;  // grid.y limit
    for (int p0 = 0; p0 < npair; p0 += chunk) {
        const int np = std::min(chunk, npair - p0);
        ra<<<dim3(nrb, np), Tr, sr, ctx->stream>>>(G, tw1, a, Z + (size_t)p0 * n0 * n1, p0);
        launched(ctx);
        cb<<<dim3(ncb, np), Tc, sc, ctx->stream>>>(G, tw0, a, Z + (size_t)p0 * n0 * n1, p0);
        launched(ctx);
        rc<<<dim3(nrb, np), Tr, sr, ctx->stream>>>(G, tw1, a, Z + (size_t)p0 * n0 * n1, p0, part);
        launched(ctx);
    }
    if (a.dots) {
        k_f2_dots<<<cdiv(2 * a.n, 256), 256, 0, ctx->stream>>>(a.n, nrb, part, a.active, a.dots);
        launched(ctx);
    }
    return true;
}

// The fused cluster kernel (fft2c.cu) + the ordered dot reduction.
static bool launch_fft2d_fused(acp_context* ctx, const FopArgs& a) {
    if (!use_f2c(ctx) || (a.mult == nullptr && a.sym < 0)) return false;
    const int npair = (a.n + 1) / 2, cs = f2c_items_per_phase(ctx->n[0]);
    double2* S = static_cast<double2*>(ctx->ws(f2_name("f2c_S", ctx->f2_alt), f2c_scratch_bytes(ctx, a.n)));
    double* part = a.dots ? ctx->wsd(f2_name("f2_part", ctx->f2_alt), (size_t)npair * cs * 4) : nullptr;
    int* q = ctx->wsi(f2_name("f2c_q", ctx->f2_alt), f2c_queue_ints(a.n));
    launch_f2c(ctx, a, S, q, part, ctx->d_twf2c);
    if (a.dots) {
        k_f2_dots<<<cdiv(2 * a.n, 256), 256, 0, ctx->stream>>>(a.n, cs, part, a.active, a.dots);
        launched(ctx);
    }
    return true;
}

void fourier_op(acp_context* ctx, const FopArgs& a) {
    if (a.n <= 0) return;
    if (ctx->dim == 2 && launch_fft2d_fused(ctx, a)) return;
    if (ctx->dim == 2 && launch_fft2d_passes(ctx, a)) return;
    IoArgs io;
    io.f = a;
    io.n = a.n;
    launch_fft<IO_OP>(ctx, io, a.n);
}

void ifft_hermitian(acp_context* ctx, const double2* spec, int n, double* out) {
    // (1/Omega) sum_k c_k e^{ikr} = (N/Omega) * (1/N) sum ...  -> scale = 1/Omega
    IoArgs io;
    io.spec = spec;
    io.out = out;
    io.n = n;
    io.scale = 1.0 / ctx->Omega;
    launch_fft<IO_HERM>(ctx, io, n);
}

void real_spectrum(acp_context* ctx, const double* x, double2* out) {
    IoArgs io;
    io.x = x;
    io.sout = out;
    io.n = 1;
    launch_fft<IO_SPEC>(ctx, io, 1);
}

// ---- multipliers ----------------------------------------------------------
__global__ void k_make_mult(int N, const double* __restrict__ k2, const double* __restrict__ khat, int kind,
                            double tau, double* __restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    double m = 0.0;
    if (kind == MULT_KINETIC) m = 0.5 * k2[i];
    else if (kind == MULT_YUKAWA) m = khat[i];
    else if (kind == MULT_PRECOND) m = 1.0 / (0.5 * k2[i] + tau);
    out[i] = m / (double)N;
}

const double* multiplier(acp_context* ctx, MultKind kind, double tau) {
    if (kind == MULT_NONE) return nullptr;
    const int N = ctx->Ng;
    std::string name = "mult" + std::to_string((int)kind);
    double* m = ctx->wsd(name, N);
    k_make_mult<<<cdiv(N, 256), 256, 0, ctx->stream>>>(N, ctx->d_k2, ctx->d_khat, (int)kind, tau, m);
    launched(ctx);
    return m;
}

// ---- model spectra ----------------------------------------------------------
// Frequency integer m of FFT bin i (numpy fftfreq order).
__device__ __forceinline__ int bin_freq(int i, int N) { return (i < (N + 1) / 2) ? i : i - N; }

// Phase e^{-i k.R} of bin (i0, i1) for position R (d components), as (cos, sin).
__device__ __forceinline__ void bin_phase(int i0, int i1, int n0, int n1, double L0, double L1, int dim,
                                          const double* R, double& c, double& s) {
    double t = (double)bin_freq(i0, n0) * R[0] / L0;
    if (dim == 2) t += (double)bin_freq(i1, n1) * R[1] / L1;
    t -= rint(t);  // exact reduction of the turn count keeps sincospi accurate
    sincospi(-2.0 * t, &s, &c);
}

// spec_{I*d+a}(k) = -i k_a Khat(k) mhat(k) e^{-i k.R_I},  mhat = -Z e^{-sigma^2 |k|^2 / 2}
__global__ void k_spectrum_G(int n0, int n1, int dim, double L0, double L1, const double* __restrict__ khat,
                             const double* __restrict__ k2, const double* __restrict__ kodd0,
                             const double* __restrict__ kodd1, double Z, double sigma,
                             const double* __restrict__ R, int NA, double2* __restrict__ spec) {
    const int N = n0 * n1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int I = blockIdx.y;
    if (i >= N || I >= NA) return;
    const int i0 = i / n1, i1 = i - i0 * n1;
    const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
    double s, c;
    bin_phase(i0, i1, n0, n1, L0, L1, dim, R + (size_t)I * dim, c, s);
    const double amp = khat[i] * mh;
    for (int a = 0; a < dim; ++a) {
        // -i k_a (c + i s) = k_a (s - i c)
        const double ka = (a == 0 ? kodd0[i0] : kodd1[i1]) * amp;
        spec[(size_t)(I * dim + a) * N + i] = make_double2(ka * s, -ka * c);
    }
}

__global__ void k_spectrum_m(int n0, int n1, int dim, double L0, double L1, const double* __restrict__ k2, double Z,
                             double sigma, const double* __restrict__ R, int NA, double2* __restrict__ spec) {
    const int N = n0 * n1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int i0 = i / n1, i1 = i - i0 * n1;
    const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
    double re = 0.0, im = 0.0;
    for (int I = 0; I < NA; ++I) {
        double s, c;
        bin_phase(i0, i1, n0, n1, L0, L1, dim, R + (size_t)I * dim, c, s);
        re += mh * c;
        im += mh * s;
    }
    spec[i] = make_double2(re, im);
}

void spectrum_G(acp_context* ctx, const double* d_R, double2* spec) {
    const int N = ctx->Ng;
    dim3 grid(cdiv(N, 256), ctx->sys.n_atoms);
    k_spectrum_G<<<grid, 256, 0, ctx->stream>>>(ctx->n[0], ctx->n[1], ctx->dim, ctx->sys.cell[0], ctx->sys.cell[1],
                                                ctx->d_khat, ctx->d_k2, ctx->d_kaxodd[0],
                                                ctx->dim == 2 ? ctx->d_kaxodd[1] : ctx->d_kaxodd[0], ctx->sys.Z,
                                                ctx->sys.sigma, d_R, ctx->sys.n_atoms, spec);
    launched(ctx);
}

void spectrum_m(acp_context* ctx, const double* d_R, double2* spec) {
    const int N = ctx->Ng;
    k_spectrum_m<<<cdiv(N, 256), 256, 0, ctx->stream>>>(ctx->n[0], ctx->n[1], ctx->dim, ctx->sys.cell[0],
                                                        ctx->sys.cell[1], ctx->d_k2, ctx->sys.Z, ctx->sys.sigma,
                                                        d_R, ctx->sys.n_atoms, spec);
    launched(ctx);
}

// ---- plan / symbol setup ---------------------------------------------------
// Per-pass twiddle tables of a plan: pass q (radix R, Ns) stores w = exp(-2 pi i r k / (Ns R))
// at twoff[q] + k (R - 1) + r - 1 (k < Ns, 1 <= r < R), argument reduced exactly in long double.
static std::vector<double2> twiddle_table(const FftPlan& pl) {
    std::vector<double2> t(pl.twoff[pl.npass] > 0 ? pl.twoff[pl.npass] : 1);
    int Ns = 1;
    for (int q = 0; q < pl.npass; ++q) {
        const int R = pl.radix[q];
        for (int k = 0; k < Ns; ++k)
            for (int r = 1; r < R; ++r) {
                const long long num = (long long)r * k, den = (long long)Ns * R;
                const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)(num % den) /
                                        (long double)den;
                t[pl.twoff[q] + k * (R - 1) + r - 1] = make_double2((double)cosl(ang), (double)sinl(ang));
            }
        Ns *= R;
    }
    return t;
}

template <class T>
static T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    ACP_CUDA(cudaMalloc(&d, v.size() * sizeof(T)));
    ACP_CUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return d;
}

static int ept_for(int E, int T) {
    const int need = (E + T - 1) / T;
    return need <= 2 ? 2 : need <= 4 ? 4 : need <= 8 ? 8 : need <= 12 ? 12 : need <= 16 ? 16 : 0;
}

void fft_init(acp_context* ctx) {
    const int dim = ctx->dim;
    ctx->n[0] = ctx->sys.grid[0];
    ctx->n[1] = dim == 2 ? ctx->sys.grid[1] : 1;
    const int n0 = ctx->n[0], n1 = ctx->n[1];
    const int N = n0 * n1;
    ctx->plan = make_plan(n0);
    if (dim == 2) ctx->plan1 = make_plan(n1);
    ctx->d_tw = upload(twiddle_table(ctx->plan));
    if (dim == 2) ctx->d_tw1 = upload(twiddle_table(ctx->plan1));
    if (dim == 2 && f2c_supported(n0, n1)) {
        std::vector<double2> t(n0);
        for (int j = 0; j < n0; ++j) {
            const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)j / (long double)n0;
            t[j] = make_double2((double)cosl(ang), (double)sinl(ang));
        }
        ctx->d_twf2c = upload(t);
    }
    // per-axis frequencies and the N_g tables (bins in C order)
    std::vector<double> kax[2], kodd[2];
    for (int a = 0; a < dim; ++a) {
        const int na = ctx->n[a];
        const double L = ctx->sys.cell[a];
        for (int i = 0; i < na; ++i) {
            const int m = (i < (na + 1) / 2) ? i : i - na;
            const double k = 2.0 * M_PI * (double)m / L;
            kax[a].push_back(k);
            kodd[a].push_back((na % 2 == 0 && i == na / 2) ? 0.0 : k);
        }
        ctx->d_kax[a] = upload(kax[a]);
        ctx->d_kaxodd[a] = upload(kodd[a]);
    }
    ctx->d_kfull = ctx->d_kax[0];
    ctx->d_kodd = ctx->d_kaxodd[0];
    std::vector<double> k2(N), khat(N);
    for (int i0 = 0; i0 < n0; ++i0)
        for (int i1 = 0; i1 < n1; ++i1) {
            double q = kax[0][i0] * kax[0][i0];
            if (dim == 2) q += kax[1][i1] * kax[1][i1];
            k2[(size_t)i0 * n1 + i1] = q;
            khat[(size_t)i0 * n1 + i1] = 4.0 * M_PI / (ctx->sys.eps0 * (q + ctx->sys.kappa * ctx->sys.kappa));
        }
    ctx->d_k2 = upload(k2);
    ctx->d_khat = upload(khat);
    // Launch geometry of the FFT kernels.  The FFT is latency-bound (log N dependent passes
    // with a block barrier each), so each CTA gets as many threads as there are radix-2
    // butterflies (<= 1024): every thread holds <= 2-4 values per pass and the chain is short.
    auto round32 = [](int t) { return (t + 31) / 32 * 32; };
    if (dim == 1) {
        // T = N/8 (<= 8 values per thread): with the register-resident inputs this keeps ~100
        // registers/thread and 4 CTAs per SM (k1_sweep on B200: 160 threads best for N = 1280)
        int T = round32((N + 7) / 8);
        T = T < 64 ? 64 : T > 1024 ? 1024 : T;
        ctx->fthreads = T;
        ctx->fept = ept_for(N, T);
        ACP_REQUIRE(ctx->fept > 0, "1D grid too large for the shared-memory FFT");
        ctx->fsmem = (size_t)padded(N) * sizeof(double2) + (size_t)N * sizeof(double);  // twiddles via L1
        // compiled-length FFT when the plan's radix schedule equals the compiled one
        auto same = [&](const int* r, int nr) {
            if (ctx->plan.npass != nr) return false;
            for (int q = 0; q < nr; ++q)
                if (ctx->plan.radix[q] != r[q]) return false;
            return true;
        };
        ctx->fct = !getenv("ACP_FFT_GENERIC") &&
                   ((N == 1280 && same(CtRadices<1280>::r, 4)) || (N == 5120 && same(CtRadices<5120>::r, 5)) ||
                    (N == 960 && same(CtRadices<960>::r, 4)) || (N == 256 && same(CtRadices<256>::r, 3)));
        ACP_REQUIRE(ctx->fsmem <= 220 * 1024, "1D grid too large for the shared-memory FFT");
    } else {
        auto same2 = [&](const FftPlan& pl, const int* r, int nr) {
            if (pl.npass != nr) return false;
            for (int q = 0; q < nr; ++q)
                if (pl.radix[q] != r[q]) return false;
            return true;
        };
        ctx->fct = !getenv("ACP_FFT_GENERIC") && n0 == n1 &&
                   ((n0 == 192 && same2(ctx->plan, CtRadices<192>::r, 3) && same2(ctx->plan1, CtRadices<192>::r, 3)) ||
                    (n0 == 256 && same2(ctx->plan, CtRadices<256>::r, 3) && same2(ctx->plan1, CtRadices<256>::r, 3)));
        // smallest cluster (cs | n0, cs | n1, cs <= 16) whose per-CTA slice has <= 4096 points
        auto slice = [&](int c) { return std::max((n0 / c) * n1, (n1 / c) * (n0 + 8)); };
        auto bytes = [&](int c) {
            return (size_t)(padded(slice(c)) + ctx->plan.twoff[ctx->plan.npass] + ctx->plan1.twoff[ctx->plan1.npass]) *
                   sizeof(double2);
        };
        int cs = 1;
        while (cs < 16 && slice(cs) > 4096 && n0 % (2 * cs) == 0 && n1 % (2 * cs) == 0) cs *= 2;
        // test knob: ACP_FFT2D_CS forces another cluster size (exercises the DSMEM transposes on small grids)
        if (const char* e = getenv("ACP_FFT2D_CS")) {
            const int f = atoi(e);
            if (f >= 1 && f <= 16 && n0 % f == 0 && n1 % f == 0) cs = f;
        }
        ACP_REQUIRE(n0 % cs == 0 && n1 % cs == 0, "2D grid not divisible by the cluster size");
        ACP_REQUIRE(bytes(cs) <= 220 * 1024, "2D grid too large for a 16-CTA cluster FFT");
        ctx->cs = cs;
        ctx->r0 = n0 / cs;
        ctx->c1 = n1 / cs;
        const int E = std::max(ctx->r0 * n1, ctx->c1 * n0);
        auto geom_for = [&](int np, int& T, int& ept, size_t& smem) {
            T = round32((np * E + 7) / 8);  // E/8 per pair (measured best in round 1)
            T = T < 64 ? 64 : T > 1024 ? 1024 : T;
            ept = ept_for(np * E, T);
            const int slice = std::max(ctx->r0 * n1, ctx->c1 * (n0 + 8));
            smem = (size_t)(padded(np * slice) + ctx->plan.twoff[ctx->plan.npass] + ctx->plan1.twoff[ctx->plan1.npass]) *
                   sizeof(double2);
        };
        // operator launches: up to NPMAX pairs per cluster while <= 8 values per thread fit
        // 1024 threads and the slices fit ~200 KB (amortises barriers and DSMEM latency)
        // Default np = 1: on B200 two pairs per cluster (1 CTA/SM) ran slower than one pair at
        // 2-3 CTAs/SM (configs[3] grid, 512 columns: 923 vs 642 us) -- occupancy beats barrier
        // amortisation here.
        int np = 1;
        ctx->fnp = np;
        geom_for(np, ctx->fthreads, ctx->fept, ctx->fsmem);
        ACP_REQUIRE(ctx->fept > 0, "2D slice too large for the FFT engine");
        geom_for(1, ctx->fthreads1, ctx->fept1, ctx->fsmem1);
    }
}

void fft_free(acp_context* ctx) {
    cudaFree(ctx->d_tw);
    cudaFree(ctx->d_tw1);
    cudaFree(ctx->d_twf2c);
    cudaFree(ctx->d_k2);
    cudaFree(ctx->d_khat);
    for (int a = 0; a < 2; ++a) {
        cudaFree(ctx->d_kax[a]);
        cudaFree(ctx->d_kaxodd[a]);
    }
}

}  // namespace acp
