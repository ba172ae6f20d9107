// fft_engine.cuh -- in-place, batched fp64 Stockham FFT in shared memory (sm_100a).
//
// Used by the 1D Fourier operator (one CTA per column pair) and the 2D operator (a
// thread-block cluster per column pair, rows / columns exchanged through DSMEM).
// A pass of radix R over `nb` independent transforms of length L stored back to back:
// every thread first loads ALL of its butterflies into registers (at most EPT complex
// values per thread), the block synchronises, then writes the results into the SAME
// buffer -- the set of locations read equals the set written, so one buffer suffices
// (half the shared memory of a ping-pong Stockham).  Twiddles exp(-2 pi i m / L) come
// from a shared-memory table.
#pragma once

#include "common.cuh"

namespace acp {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }  // * (-i)

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

// Shared-memory index padding: one spare 16-byte slot every 8 complex values.  A 16-byte
// access touches 4 banks, so 8 consecutive values fill all 32 banks; the first Stockham pass
// writes with stride R (and the 2D transposes with stride ld), which without padding puts 8
// lanes of a quarter-warp on the same 4 banks.  With the pad every pattern here is
// conflict-free (checked by enumeration for the c1 / 2D plans).
__device__ __forceinline__ int P(int i) { return i + (i >> 3); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 3) + 1; }

// Twiddles: one table per Stockham pass, laid out [k][r-1] for the pass's Ns sub-transform
// offsets k and radix digits r = 1..R-1: w = exp(-2 pi i r k / (Ns R)), each entry correctly
// rounded on the host.  A butterfly reads its R-1 twiddles contiguously (stride R-1 across
// threads, odd for R = 8, 4, 2: conflict-free) -- no power recurrences, no 2-level products.
// FftPlan::twoff[p] is pass p's offset; FftPlan::twoff[npass] the table length.

// q = floor(a / d) for 0 <= a < 2^21, d >= 1, via a float reciprocal: (a + 0.5)/d lies at least
// 0.5/d from an integer, and the two roundings of (a + 0.5) * fl(1/d) err by < 2^-22 (a + 0.5)/d
// < 0.5/d.  Avoids the ~20-instruction integer division.
__device__ __forceinline__ int fdiv(int a, float rd) { return __float2int_rz(((float)a + 0.5f) * rd); }

// One in-place Stockham pass of radix R over nb transforms of length L (transform t at buf + t*ld,
// padded indexing P): sub-transforms of length Ns are combined into length Ns*R.  EPT = max
// complex values a thread holds (EPT >= nb*L / blockDim.x).  Ends with a block barrier.
template <int R, int EPT>
__device__ __forceinline__ void pass_inplace(double2* buf, int L, int ld, int nb, int Ns, const double2* __restrict__ tw) {
    constexpr int MB = (EPT + R - 1) / R;
    const int per = L / R;              // butterflies per transform
    const int total = nb * per;
    const float rper = 1.0f / (float)per, rNs = 1.0f / (float)Ns;
    double2 x[MB][R];
#pragma unroll
    for (int b = 0; b < MB; ++b) {
        const int g = threadIdx.x + b * blockDim.x;
        if (g < total) {
            const int t = nb == 1 ? 0 : fdiv(g, rper);
            const int j = g - t * per;
            const int k = j - Ns * fdiv(j, rNs);
            const int base = t * ld + j;
#pragma unroll
            for (int r = 0; r < R; ++r) x[b][r] = buf[P(base + r * per)];
            if (Ns > 1) {
                const double2* tk = tw + k * (R - 1);
#pragma unroll
                for (int r = 1; r < R; ++r) x[b][r] = cmul(x[b][r], tk[r - 1]);
            }
            dft<R>(x[b]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < MB; ++b) {
        const int g = threadIdx.x + b * blockDim.x;
        if (g < total) {
            const int t = nb == 1 ? 0 : fdiv(g, rper);
            const int j = g - t * per;
            const int k = j - Ns * fdiv(j, rNs);
            const int base = t * ld + (j - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) buf[P(base + r * Ns)] = x[b][r];
        }
    }
    __syncthreads();
}

// Compile-time Stockham pass over NB transforms of length L (transform t at buf + t*LD; NB = 1
// for the 1D kernels): the same data movement and arithmetic as pass_inplace, but every index is
// a constant expression of the butterfly index, and strides that are multiples of 8 make the
// padded index linear in r (P(b + r s) = P(b) + r (s + s/8)), so an element costs an immediate
// offset instead of a pad computation.
template <int R, int L, int NS, int NB, int LD, int EPT>
__device__ __forceinline__ void pass_ct(double2* buf, const double2* __restrict__ tw) {
    constexpr int PER = L / R;
    constexpr int TOTAL = NB * PER;
    constexpr int MB = (EPT + R - 1) / R;
    constexpr bool LIN_LD = PER % 8 == 0 && (NB == 1 || LD % 8 == 0);
    double2 x[MB][R];
#pragma unroll
    for (int b = 0; b < MB; ++b) {
        const int g = threadIdx.x + b * blockDim.x;
        if (g < TOTAL) {
            const int t = NB == 1 ? 0 : g / PER;
            const int j = g - t * PER;
            const int base = t * LD + j;
            if constexpr (LIN_LD) {
                const int pb = P(base);
#pragma unroll
                for (int r = 0; r < R; ++r) x[b][r] = buf[pb + r * (PER + PER / 8)];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) x[b][r] = buf[P(base + r * PER)];
            }
            if constexpr (NS > 1) {
                const double2* tk = tw + (j % NS) * (R - 1);
#pragma unroll
                for (int r = 1; r < R; ++r) x[b][r] = cmul(x[b][r], tk[r - 1]);
            }
            dft<R>(x[b]);
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < MB; ++b) {
        const int g = threadIdx.x + b * blockDim.x;
        if (g < TOTAL) {
            const int t = NB == 1 ? 0 : g / PER;
            const int j = g - t * PER;
            const int k = j % NS;
            const int b2 = t * LD + (j - k) * R + k;
            if constexpr (NS % 8 == 0 && (NB == 1 || LD % 8 == 0)) {
                const int pb = P(b2);
#pragma unroll
                for (int r = 0; r < R; ++r) buf[pb + r * (NS + NS / 8)] = x[b][r];
            } else if constexpr (NS == 1 && R == 8 && (NB == 1 || LD % 8 == 0)) {
                const int pb = P(b2);  // b2 = t LD + 8 j: the 8 outputs share one pad block
#pragma unroll
                for (int r = 0; r < R; ++r) buf[pb + r] = x[b][r];
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) buf[P(b2 + r * NS)] = x[b][r];
            }
        }
    }
    __syncthreads();
}

template <int EPT, int L, int NB, int LD, int NS, int OFF, int R, int... Rs>
__device__ __forceinline__ void fft_ct_passes(double2* buf, const double2* __restrict__ tw) {
    pass_ct<R, L, NS, NB, LD, EPT>(buf, tw + OFF);
    if constexpr (sizeof...(Rs) > 0) fft_ct_passes<EPT, L, NB, LD, NS * R, OFF + NS * (R - 1), Rs...>(buf, tw);
}

// Radix schedules of the compiled lengths -- identical to make_plan's (8s, then 4, 2, 5, 3),
// which the host checks before selecting a compiled kernel (the twiddle tables follow the plan).
template <int N> struct CtRadices;
template <> struct CtRadices<1280> { static constexpr int r[] = {8, 8, 4, 5}; };
template <> struct CtRadices<5120> { static constexpr int r[] = {8, 8, 8, 2, 5}; };
template <> struct CtRadices<960> { static constexpr int r[] = {8, 8, 5, 3}; };
template <> struct CtRadices<256> { static constexpr int r[] = {8, 8, 4}; };
template <> struct CtRadices<192> { static constexpr int r[] = {8, 8, 3}; };

// NB transforms of the compiled length N at stride LD (NB = 1: one transform, LD unused).
template <int N, int EPT, int NB = 1, int LD = 0>
__device__ __forceinline__ void fft_ct(double2* buf, const double2* __restrict__ tw) {
    if constexpr (N == 1280) fft_ct_passes<EPT, 1280, NB, LD, 1, 0, 8, 8, 4, 5>(buf, tw);
    else if constexpr (N == 5120) fft_ct_passes<EPT, 5120, NB, LD, 1, 0, 8, 8, 8, 2, 5>(buf, tw);
    else if constexpr (N == 960) fft_ct_passes<EPT, 960, NB, LD, 1, 0, 8, 8, 5, 3>(buf, tw);
    else if constexpr (N == 256) fft_ct_passes<EPT, 256, NB, LD, 1, 0, 8, 8, 4>(buf, tw);
    else if constexpr (N == 192) fft_ct_passes<EPT, 192, NB, LD, 1, 0, 8, 8, 3>(buf, tw);
}

// Forward FFT (exp(-i ...)) of nb transforms of length pl.N in place (transform t at buf + t*ld).
template <int EPT>
__device__ __forceinline__ void fft_inplace(double2* buf, int ld, int nb, const FftPlan& pl,
                                            const double2* __restrict__ tw) {
    // The plan lists its radices in the fixed order 8, 4, 2, 5, 3 (make_plan); one loop per
    // radix keeps the register allocation of each pass independent (a switch inside a single
    // loop made ptxas keep every variant's butterfly registers live at once).
    int Ns = 1, p = 0;
    for (; p < pl.npass && pl.radix[p] == 8; ++p, Ns *= 8) pass_inplace<8, EPT>(buf, pl.N, ld, nb, Ns, tw + pl.twoff[p]);
    for (; p < pl.npass && pl.radix[p] == 4; ++p, Ns *= 4) pass_inplace<4, EPT>(buf, pl.N, ld, nb, Ns, tw + pl.twoff[p]);
    for (; p < pl.npass && pl.radix[p] == 2; ++p, Ns *= 2) pass_inplace<2, EPT>(buf, pl.N, ld, nb, Ns, tw + pl.twoff[p]);
    for (; p < pl.npass && pl.radix[p] == 5; ++p, Ns *= 5) pass_inplace<5, EPT>(buf, pl.N, ld, nb, Ns, tw + pl.twoff[p]);
    for (; p < pl.npass && pl.radix[p] == 3; ++p, Ns *= 3) pass_inplace<3, EPT>(buf, pl.N, ld, nb, Ns, tw + pl.twoff[p]);
}

// Copy a plan's twiddle table (pl.twoff[pl.npass] entries) into shared memory with cp.async
// (16-byte chunks, no register round trip: the copies overlap whatever the CTA does next).
// The caller commits/waits and synchronises before the first twiddled pass.
__device__ __forceinline__ void cp_async16_fe(void* smem, const void* gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all_fe() {
    asm volatile("cp.async.commit_group;\n" ::);
    asm volatile("cp.async.wait_group 0;\n" ::);
}
__device__ __forceinline__ const double2* load_twiddles(double2* dst, const double2* __restrict__ src,
                                                        const FftPlan& pl) {
    const int n = pl.twoff[pl.npass];
    for (int i = threadIdx.x; i < n; i += blockDim.x) cp_async16_fe(dst + i, src + i);
    return dst;
}

// Deterministic block sum of 4 values (fixed reduction tree); red needs 132 doubles.
__device__ __forceinline__ void block_sum4(double* v, double* red) {
#pragma unroll
    for (int q = 0; q < 4; ++q)
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
    __syncthreads();
    if (l == 0)
#pragma unroll
        for (int q = 0; q < 4; ++q) red[4 * w + q] = v[q];
    __syncthreads();
    if (threadIdx.x < 4) {
        double s = 0.0;
        for (int i = 0; i < nw; ++i) s += red[4 * i + threadIdx.x];
        red[128 + threadIdx.x] = s;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = red[128 + q];
}

}  // namespace acp
