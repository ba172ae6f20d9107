// fft.cu -- in-house fp64 FFT in shared memory and the Fourier-operator kernel (K1).
//
// The Hamiltonian apply of PAPER.md:189 (Eq. Hamil), H psi = -1/2 Delta psi + V psi,
// uses the Fourier symbol |k|^2/2 for -1/2 Delta on the periodic grid (PAPER.md:852
// "plane wave basis set").  One CTA transforms one PAIR of real columns packed as
// z = a + i b (Hermitian multipliers keep the two results separable), with a
// Stockham autosort FFT (radices 8/4/2/5/3) ping-ponging between two shared-memory
// buffers; the pointwise (V - shift) multiply, the multiplier and the per-column
// dot products are fused into the same pass, so each column is read once and
// written once from HBM.
#include "common.cuh"

#include <cmath>

namespace acp {

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
    return p;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// multiply by -i
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }

// Forward DFTs of small radix, in registers: y_s = sum_r x_r exp(-2 pi i r s / R).
template <int R> __device__ __forceinline__ void dft(double2* x);

template <> __device__ __forceinline__ void dft<2>(double2* x) {
    double2 a = x[0], b = x[1];
    x[0] = cadd(a, b);
    x[1] = csub(a, b);
}
template <> __device__ __forceinline__ void dft<4>(double2* x) {
    double2 t0 = cadd(x[0], x[2]), t1 = csub(x[0], x[2]);
    double2 t2 = cadd(x[1], x[3]), t3 = mul_mi(csub(x[1], x[3]));
    x[0] = cadd(t0, t2);
    x[2] = csub(t0, t2);
    x[1] = cadd(t1, t3);
    x[3] = csub(t1, t3);
}
template <> __device__ __forceinline__ void dft<8>(double2* x) {
    double2 e[4] = {x[0], x[2], x[4], x[6]};
    double2 o[4] = {x[1], x[3], x[5], x[7]};
    dft<4>(e);
    dft<4>(o);
    const double h = 0.70710678118654752440;  // sqrt(1/2)
    // w8^k = exp(-i pi k / 4)
    double2 o1 = make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    double2 o2 = mul_mi(o[2]);
    double2 o3 = make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
    x[0] = cadd(e[0], o[0]);
    x[4] = csub(e[0], o[0]);
    x[1] = cadd(e[1], o1);
    x[5] = csub(e[1], o1);
    x[2] = cadd(e[2], o2);
    x[6] = csub(e[2], o2);
    x[3] = cadd(e[3], o3);
    x[7] = csub(e[3], o3);
}
template <> __device__ __forceinline__ void dft<3>(double2* x) {
    const double s1 = 0.86602540378443864676;  // sin(2 pi / 3)
    double2 a = cadd(x[1], x[2]);
    double2 b = csub(x[1], x[2]);
    double2 y0 = cadd(x[0], a);
    double2 t = make_double2(x[0].x - 0.5 * a.x, x[0].y - 0.5 * a.y);
    double2 u = make_double2(s1 * b.y, -s1 * b.x);  // -i s1 b
    x[0] = y0;
    x[1] = cadd(t, u);
    x[2] = csub(t, u);
}
template <> __device__ __forceinline__ void dft<5>(double2* x) {
    const double c1 = 0.30901699437494742410;   // cos(2 pi/5)
    const double c2 = -0.80901699437494742410;  // cos(4 pi/5)
    const double s1 = 0.95105651629515357212;   // sin(2 pi/5)
    const double s2 = 0.58778525229247312917;   // sin(4 pi/5)
    double2 a1 = cadd(x[1], x[4]), b1 = csub(x[1], x[4]);
    double2 a2 = cadd(x[2], x[3]), b2 = csub(x[2], x[3]);
    double2 y0 = make_double2(x[0].x + a1.x + a2.x, x[0].y + a1.y + a2.y);
    double2 t1 = make_double2(x[0].x + c1 * a1.x + c2 * a2.x, x[0].y + c1 * a1.y + c2 * a2.y);
    double2 t2 = make_double2(x[0].x + c2 * a1.x + c1 * a2.x, x[0].y + c2 * a1.y + c1 * a2.y);
    double2 u1 = make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
    double2 u2 = make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
    x[0] = y0;
    x[1] = cadd(t1, mul_mi(u1));
    x[4] = csub(t1, mul_mi(u1));
    x[2] = cadd(t2, mul_mi(u2));
    x[3] = csub(t2, mul_mi(u2));
}

// One Stockham pass of radix R: sub-transforms of length Ns are combined into
// length Ns*R; input read with stride N/R, output written in natural order.
template <int R>
__device__ __forceinline__ void stockham_pass(const double2* __restrict__ src, double2* __restrict__ dst,
                                              int N, int Ns, const double2* __restrict__ tw) {
    const int nb = N / R;
    const int stride = N / (Ns * R);
    for (int j = threadIdx.x; j < nb; j += blockDim.x) {
        const int k = j % Ns;
        double2 x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = src[j + r * nb];
        if (Ns > 1) {
#pragma unroll
            for (int r = 1; r < R; ++r) x[r] = cmul(x[r], __ldg(&tw[r * k * stride]));
        }
        dft<R>(x);
        const int base = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < R; ++r) dst[base + r * Ns] = x[r];
    }
}

// Forward FFT of a (length N) using b as scratch; returns the buffer holding the result.
__device__ double2* fft_forward(double2* a, double2* b, const FftPlan& pl, const double2* __restrict__ tw) {
    double2* src = a;
    double2* dst = b;
    int Ns = 1;
    for (int p = 0; p < pl.npass; ++p) {
        const int R = pl.radix[p];
        switch (R) {
            case 8: stockham_pass<8>(src, dst, pl.N, Ns, tw); break;
            case 4: stockham_pass<4>(src, dst, pl.N, Ns, tw); break;
            case 2: stockham_pass<2>(src, dst, pl.N, Ns, tw); break;
            case 5: stockham_pass<5>(src, dst, pl.N, Ns, tw); break;
            default: stockham_pass<3>(src, dst, pl.N, Ns, tw); break;
        }
        __syncthreads();
        double2* t = src;
        src = dst;
        dst = t;
        Ns *= R;
    }
    return src;
}

// Deterministic block sum of up to 2 values (fixed reduction tree).
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0) {
        red[2 * w] = a;
        red[2 * w + 1] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double s0 = 0.0, s1 = 0.0;
        for (int i = 0; i < nw; ++i) {
            s0 += red[2 * i];
            s1 += red[2 * i + 1];
        }
        red[0] = s0;
        red[1] = s1;
    }
    __syncthreads();
    a = red[0];
    b = red[1];
}

// K1: Y = IFFT(mult . FFT(X)) + (diag - shift_j) X for the column pair (2 blockIdx.x, +1).
__global__ void __launch_bounds__(256) k_fourier_op(FftPlan pl, const double2* __restrict__ tw, FopArgs a) {
    extern __shared__ double2 smem[];
    const int N = pl.N;
    double2* b0 = smem;
    double2* b1 = smem + N;
    __shared__ double red[2 * 32 + 4];
    const int c0 = 2 * blockIdx.x;
    const int c1 = c0 + 1;
    const bool has1 = c1 < a.n;
    bool act0 = true, act1 = has1;
    if (a.active) {
        act0 = a.active[c0] != 0;
        act1 = has1 && a.active[c1] != 0;
    }
    if (!act0 && !act1) return;
    const double* x0 = a.X + (size_t)c0 * N;
    const double* x1 = a.X + (size_t)c1 * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x)
        b0[i] = make_double2(x0[i], has1 ? x1[i] : 0.0);
    __syncthreads();
    double2* F = nullptr;
    if (a.mult) {
        F = fft_forward(b0, b1, pl, tw);
        // conj(mult * F) then forward FFT == N * conj(IFFT(mult * F)) (1/N folded into mult)
        for (int i = threadIdx.x; i < N; i += blockDim.x) {
            const double m = __ldg(&a.mult[i]);
            double2 v = F[i];
            F[i] = make_double2(m * v.x, -m * v.y);
        }
        __syncthreads();
        double2* other = (F == b0) ? b1 : b0;
        F = fft_forward(F, other, pl, tw);
    }
    const double s0 = a.shift ? a.shift[c0] : 0.0;
    const double s1 = (a.shift && has1) ? a.shift[c1] : 0.0;
    double d00 = 0.0, d01 = 0.0, d10 = 0.0, d11 = 0.0;
    double* y0 = a.Y + (size_t)c0 * N;
    double* y1 = a.Y + (size_t)c1 * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        const double u0 = x0[i];
        const double u1 = has1 ? x1[i] : 0.0;
        double v0 = 0.0, v1 = 0.0;
        if (F) {
            v0 = F[i].x;
            v1 = -F[i].y;
        }
        if (a.diag) {
            const double dg = a.diag[i];
            v0 += (dg - s0) * u0;
            v1 += (dg - s1) * u1;
        } else if (a.shift) {
            v0 -= s0 * u0;
            v1 -= s1 * u1;
        }
        if (act0) y0[i] = v0;
        if (act1) y1[i] = v1;
        d00 += u0 * v0;
        d01 += u0 * u0;
        d10 += u1 * v1;
        d11 += u1 * u1;
    }
    if (a.dots) {
        block_sum2(d00, d01, red);
        block_sum2(d10, d11, red);
        if (threadIdx.x == 0) {
            if (act0) {
                a.dots[2 * c0] = d00;
                a.dots[2 * c0 + 1] = d01;
            }
            if (act1) {
                a.dots[2 * c1] = d10;
                a.dots[2 * c1 + 1] = d11;
            }
        }
    }
}

static int fop_threads(int N) {
    int t = N / 8;
    if (t < 64) t = 64;
    if (t > 256) t = 256;
    return (t + 31) / 32 * 32;
}

void fourier_op(acp_context* ctx, const FopArgs& a) {
    if (a.n <= 0) return;
    const int N = ctx->plan.N;
    const size_t smem = 2 * (size_t)N * sizeof(double2);
    const int npair = (a.n + 1) / 2;
    k_fourier_op<<<npair, fop_threads(N), smem, ctx->stream>>>(ctx->plan, ctx->d_tw, a);
    launched(ctx);
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
    const int N = ctx->plan.N;
    std::string name = "mult" + std::to_string((int)kind);
    double* m = ctx->wsd(name, N);
    k_make_mult<<<cdiv(N, 256), 256, 0, ctx->stream>>>(N, ctx->d_k2, ctx->d_khat, (int)kind, tau, m);
    launched(ctx);
    return m;
}

// ---- Hermitian spectra -> real grid functions ------------------------------
// out_j(r_alpha) = (1/Omega) sum_k spec_j(k) e^{i k r_alpha}, columns packed in pairs.
__global__ void __launch_bounds__(256) k_ifft_hermitian(FftPlan pl, const double2* __restrict__ tw,
                                                        const double2* __restrict__ spec, int n,
                                                        double scale, double* __restrict__ out) {
    extern __shared__ double2 smem[];
    const int N = pl.N;
    double2* b0 = smem;
    double2* b1 = smem + N;
    const int c0 = 2 * blockIdx.x, c1 = c0 + 1;
    const bool has1 = c1 < n;
    const double2* s0 = spec + (size_t)c0 * N;
    const double2* s1 = spec + (size_t)c1 * N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        double2 p = s0[i];
        double2 q = has1 ? s1[i] : make_double2(0.0, 0.0);
        // Z = P + i Q ; load conj(Z)
        b0[i] = make_double2(p.x - q.y, -(p.y + q.x));
    }
    __syncthreads();
    double2* F = fft_forward(b0, b1, pl, tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
        out[(size_t)c0 * N + i] = F[i].x * scale;
        if (has1) out[(size_t)c1 * N + i] = -F[i].y * scale;
    }
}

void ifft_hermitian(acp_context* ctx, const double2* spec, int n, double* out) {
    const int N = ctx->plan.N;
    const size_t smem = 2 * (size_t)N * sizeof(double2);
    // (1/Omega) sum_k c_k e^{ikr} = (N/Omega) * (1/N) sum ...  -> scale = 1/Omega
    k_ifft_hermitian<<<(n + 1) / 2, fop_threads(N), smem, ctx->stream>>>(ctx->plan, ctx->d_tw, spec, n,
                                                                         1.0 / ctx->Omega, out);
    launched(ctx);
}

// Frequency integer m of FFT bin i (numpy fftfreq order).
__device__ __forceinline__ int bin_freq(int i, int N) { return (i < (N + 1) / 2) ? i : i - N; }

// spec_{I*d+a}(k) = -i k_a Khat(k) mhat(k) e^{-i k R_I},  mhat = -Z e^{-sigma^2 k^2 / 2}   (1D)
__global__ void k_spectrum_G(int N, double L, const double* __restrict__ khat, const double* __restrict__ kodd,
                             const double* __restrict__ k2, double Z, double sigma, const double* __restrict__ R,
                             int NA, double2* __restrict__ spec) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    int I = blockIdx.y;
    if (i >= N || I >= NA) return;
    const int m = bin_freq(i, N);
    const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
    double s, c;
    sincospi(-2.0 * (double)m * R[I] / L, &s, &c);  // e^{-i k R}, k = 2 pi m / L
    const double amp = khat[i] * mh;
    // -i k a (c + i s) = k a (s - i c)
    const double ka = kodd[i] * amp;
    spec[(size_t)I * N + i] = make_double2(ka * s, -ka * c);
}

__global__ void k_spectrum_m(int N, double L, const double* __restrict__ k2, double Z, double sigma,
                             const double* __restrict__ R, int NA, double2* __restrict__ spec) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const int m = bin_freq(i, N);
    const double mh = -Z * exp(-0.5 * sigma * sigma * k2[i]);
    double re = 0.0, im = 0.0;
    for (int I = 0; I < NA; ++I) {
        double s, c;
        sincospi(-2.0 * (double)m * R[I] / L, &s, &c);
        re += mh * c;
        im += mh * s;
    }
    spec[i] = make_double2(re, im);
}

void spectrum_G(acp_context* ctx, const double* d_R, double2* spec) {
    ACP_REQUIRE(ctx->dim == 1, "2D perturbations not built in this round");
    const int N = ctx->plan.N;
    dim3 grid(cdiv(N, 256), ctx->sys.n_atoms);
    k_spectrum_G<<<grid, 256, 0, ctx->stream>>>(N, ctx->sys.cell[0], ctx->d_khat, ctx->d_kodd, ctx->d_k2,
                                                ctx->sys.Z, ctx->sys.sigma, d_R, ctx->sys.n_atoms, spec);
    launched(ctx);
}

void spectrum_m(acp_context* ctx, const double* d_R, double2* spec) {
    const int N = ctx->plan.N;
    k_spectrum_m<<<cdiv(N, 256), 256, 0, ctx->stream>>>(N, ctx->sys.cell[0], ctx->d_k2, ctx->sys.Z,
                                                        ctx->sys.sigma, d_R, ctx->sys.n_atoms, spec);
    launched(ctx);
}

// Spectrum of one real column: out(k) = sum_a x(a) e^{-i k r_a}.
__global__ void __launch_bounds__(256) k_real_spectrum(FftPlan pl, const double2* __restrict__ tw,
                                                       const double* __restrict__ x, double2* __restrict__ out) {
    extern __shared__ double2 smem[];
    const int N = pl.N;
    for (int i = threadIdx.x; i < N; i += blockDim.x) smem[i] = make_double2(x[i], 0.0);
    __syncthreads();
    double2* F = fft_forward(smem, smem + N, pl, tw);
    for (int i = threadIdx.x; i < N; i += blockDim.x) out[i] = F[i];
}

void real_spectrum(acp_context* ctx, const double* x, double2* out) {
    const int N = ctx->plan.N;
    k_real_spectrum<<<1, fop_threads(N), 2 * (size_t)N * sizeof(double2), ctx->stream>>>(ctx->plan, ctx->d_tw, x, out);
    launched(ctx);
}

// ---- plan / symbol setup ---------------------------------------------------
void fft_init(acp_context* ctx) {
    ACP_REQUIRE(ctx->dim == 1, "only d = 1 grids are built in this round (2D is a later row)");
    const int N = ctx->Ng;
    ctx->plan = make_plan(N);
    std::vector<double2> tw(N);
    for (int m = 0; m < N; ++m) {
        // exact argument reduction in long double, then round
        long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)m / (long double)N;
        tw[m] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    std::vector<double> k2(N), kodd(N), kfull(N), khat(N);
    const double L = ctx->sys.cell[0];
    for (int i = 0; i < N; ++i) {
        int m = (i < (N + 1) / 2) ? i : i - N;
        double k = 2.0 * M_PI * (double)m / L;
        kfull[i] = k;
        kodd[i] = (N % 2 == 0 && i == N / 2) ? 0.0 : k;
        k2[i] = k * k;
        khat[i] = 4.0 * M_PI / (ctx->sys.eps0 * (k * k + ctx->sys.kappa * ctx->sys.kappa));
    }
    ACP_CUDA(cudaMalloc(&ctx->d_tw, N * sizeof(double2)));
    ACP_CUDA(cudaMalloc(&ctx->d_k2, N * sizeof(double)));
    ACP_CUDA(cudaMalloc(&ctx->d_kodd, N * sizeof(double)));
    ACP_CUDA(cudaMalloc(&ctx->d_kfull, N * sizeof(double)));
    ACP_CUDA(cudaMalloc(&ctx->d_khat, N * sizeof(double)));
    ACP_CUDA(cudaMemcpy(ctx->d_tw, tw.data(), N * sizeof(double2), cudaMemcpyHostToDevice));
    ACP_CUDA(cudaMemcpy(ctx->d_k2, k2.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    ACP_CUDA(cudaMemcpy(ctx->d_kodd, kodd.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    ACP_CUDA(cudaMemcpy(ctx->d_kfull, kfull.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    ACP_CUDA(cudaMemcpy(ctx->d_khat, khat.data(), N * sizeof(double), cudaMemcpyHostToDevice));
    const size_t smem = 2 * (size_t)N * sizeof(double2);
    ACP_REQUIRE(smem <= 227 * 1024, "grid too large for the shared-memory FFT");
    ACP_CUDA(cudaFuncSetAttribute(k_fourier_op, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ACP_CUDA(cudaFuncSetAttribute(k_ifft_hermitian, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    ACP_CUDA(cudaFuncSetAttribute(k_real_spectrum, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

void fft_free(acp_context* ctx) {
    cudaFree(ctx->d_tw);
    cudaFree(ctx->d_k2);
    cudaFree(ctx->d_kodd);
    cudaFree(ctx->d_kfull);
    cudaFree(ctx->d_khat);
}

}  // namespace acp
