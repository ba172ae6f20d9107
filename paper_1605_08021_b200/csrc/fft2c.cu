// fft2c.cu -- fused 2D Fourier operator (K1) for square n x n grids, n = 16 N2 (N2 = 2..16).
//
// Y = IFFT2(m . FFT2(X)) + (V - shift_j) (.) X for a batch of real columns, two columns packed
// as z = x0 + i x1 (real-even symbols keep them separable), inverse by conjugation (1/N folded
// into the symbol) -- the same operator as the three-pass kernels of fft.cu (PAPER.md:189 Eq.
// Hamil: H = -1/2 Delta + V; the CG preconditioner is the symbol 1/(|k|^2/2 + tau)).
//
// ONE persistent launch, one 256-thread CTA per SM (two for n = 192).  A column pair is three
// phases, each cut into IPP items of BPI batches; a batch is 16 one-dimensional transforms:
//   A  rows:    row FFTs of z (x read from HBM)                          -> plane S1[k1][i0]
//   B  columns: FFT, conj(m .), FFT (= conj of the inverse)              -> plane S2[i0][k1]
//   C  rows:    row FFTs of S2, unpack, + (V - shift) x, masked write, per-item partial dots
// Every batch's input is ONE contiguous block (16 rows of x0 and of x1, 16 columns of S1, 16 rows
// of S2), fetched by the Tensor Memory Accelerator (cp.async.bulk, mbarrier completion) into a
// double-buffered shared-memory stage one batch AHEAD of the compute; the block is then
// exchanged in place through the same buffer.  CTAs take items from a global atomic queue in a
// skewed order (step s: A of pair s, B of pair s - d, C of pair s - 2d), so an item's producers
// finished long before; the issuing thread checks their counter (acquire) before the prefetch.
// Items only wait on items dequeued before them, which running CTAs hold: no deadlock.  The
// planes of the pairs in flight live in a ring of R slots re-used by every pair, so the two
// transposes stay in the 126 MB L2 and only x (read) and y (written) touch HBM; x is loaded
// evict_last by A and re-read (evict_first) by C.
// Each 1D transform is two register passes with one exchange (fft2c.cuh); B's forward and
// inverse column transforms chain through registers.
#include <cstdio>

#include "common.cuh"
#include "fft2c.cuh"

// 16-line batches per queue item (A/B at build time, -DACP_F2C_BPI=n).  c4g, 38088 columns, best queue
// skew each: 1 -> 32.0 ms, 2 -> 26.94, 4 -> 25.50, 8 -> 26.1, 16 -> 28.8 (runs R5f, R5g)
// -DACP_F2C_DISCARD=m (A/B at build time): drop a consumed plane block from L2 (discard.global.L2)
// instead of letting it be written back -- 1: all threads before the batch, 2: after it, 3: one warp
// after it.  c4g, 38088 columns, m = 1: DRAM writes 59.2 -> 29.8 GB per launch but 26.07 vs 25.18 ms
// (run R6c): the kernel is not DRAM-bound, the CCTLs cost issue slots.  Default 0.
#ifndef ACP_F2C_DISCARD
#define ACP_F2C_DISCARD 0
#endif
#ifndef ACP_F2C_BPI
#define ACP_F2C_BPI 4
#endif

namespace acp {

template <int N>
struct F2C {
    static constexpr int N2 = N / 16;
    static constexpr int CS = N / 16;               // 16-line batches per phase and pair
    static constexpr int BPI = CS >= ACP_F2C_BPI ? ACP_F2C_BPI : 1;  // batches per item
    static constexpr int IPP = CS / BPI;            // items per phase and pair
    static constexpr int TB = N2 * 17 + 1;          // exchange row stride, steps 1 -> 2 (odd)
    static constexpr int TB2 = 16 * (N2 + 1) + 1;   // exchange row stride, inverse steps (odd)
    static constexpr int STAGE = 16 * N;            // staged batch input (complex entries)
    static constexpr int BUF = (16 * (TB > TB2 ? TB : TB2) > STAGE ? 16 * (TB > TB2 ? TB : TB2) : STAGE);
    static constexpr size_t SMEM = 2 * (size_t)BUF * sizeof(double2);
};

static size_t f2c_smem(int N) {
    switch (N) {
        case 32: return F2C<32>::SMEM;
        case 64: return F2C<64>::SMEM;
        case 128: return F2C<128>::SMEM;
        case 192: return F2C<192>::SMEM;
        case 256: return F2C<256>::SMEM;
    }
    return 0;
}
static int f2c_ipp(int N) { return (N / 16) / (N / 16 >= ACP_F2C_BPI ? ACP_F2C_BPI : 1); }

struct F2cArgs {
    FopArgs a;
    int N;                 // n (grid points per axis)
    int Ng;
    double dk0, dk1, invN;
    const double2* tw;     // exp(-2 pi i j / n), j < n
    double2* S;            // ring of R slots, 2 N^2 complex each (S1 then S2)
    int R;                 // ring slots
    int d;                 // queue skew (steps between A and B, B and C of a pair)
    int npair;
    int nsteps;            // npair + 2 d
    int* queue;            // [0] = next item; then cnt[3 * npair] (A, B, C done-counts per pair)
    double* part;          // per (pair, item of C): 4 partial dots
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ unsigned long long pol_first() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long pol_last() {
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// (not volatile: the compiler may batch these loads ahead of the stores -- x, V and the symbol
// table are never written inside the kernel, and y[o] is only written after x[o] was read)
__device__ __forceinline__ double ld_hint(const double* a, unsigned long long pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ double ld_nc(const double* a) {
    double v;
    asm("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(a));
    return v;
}
__device__ __forceinline__ void st_hint(double* a, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(a), "d"(v), "l"(pol));
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
// global -> shared bulk copy by the TMA engine; completion counted on the mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         unsigned long long pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n @!P bra WAIT_%=;\n}" ::"r"(
            smem_addr(bar)),
        "r"(parity)
        : "memory");
}
// threads' generic-proxy accesses of shared memory happen-before later bulk (async-proxy) writes
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }


// ---------------------------------------------------------------- work items
struct Item {
    int p, phase, q;   // pair, phase (0 A, 1 B, 2 C), item within the phase
    int skip;          // 0: work; 1: pair inactive (count only); 2: out of range (nothing)
};

template <int N>
__device__ __forceinline__ Item decode(const F2cArgs& g, int item) {
    constexpr int IPP = F2C<N>::IPP;
    Item it;
    const int total = g.nsteps * 3 * IPP;
    if (item >= total) {
        it.p = -1;
        it.phase = 0;
        it.q = 0;
        it.skip = 3;  // end of queue
        return it;
    }
    const int step = item / (3 * IPP), rem = item - step * 3 * IPP;
    it.phase = rem / IPP;
    it.q = rem - it.phase * IPP;
    it.p = step - it.phase * g.d;
    it.skip = 0;
    if (it.p < 0 || it.p >= g.npair) {
        it.skip = 2;
        return it;
    }
    const FopArgs& a = g.a;
    const int c0 = 2 * it.p;
    const bool h1 = c0 + 1 < a.n;
    if (a.active && !a.active[c0] && !(h1 && a.active[c0 + 1])) it.skip = 1;
    return it;
}

// Producers of item `it` are done and its ring slot is free (checked once, before batch 0).
// block = false: one look, no waiting (the one-ahead prefetch must never wait while this CTA still
// holds an unfinished item -- the item it would wait for may be that very item).
template <int N>
__device__ __forceinline__ bool deps_ready(const F2cArgs& g, const Item& it, bool block) {
    using K = F2C<N>;
    const int* cnt = g.queue + 1;
    const int p = it.p;
    const int* w[2] = {nullptr, nullptr};
    if (it.phase == 0 && p >= g.R) w[0] = &cnt[3 * (p - g.R) + 1];   // old pair's B read S1
    if (it.phase == 1) {
        w[0] = &cnt[3 * p + 0];                                      // all rows of the pair
        if (p >= g.R) w[1] = &cnt[3 * (p - g.R) + 2];                // old pair's C read S2
    }
    if (it.phase == 2) w[0] = &cnt[3 * p + 1];                       // all columns of the pair
    for (int i = 0; i < 2; ++i) {
        if (!w[i]) continue;
        if (!block) {
            if (ld_acquire(w[i]) < K::IPP) return false;
        } else {
            while (ld_acquire(w[i]) < K::IPP) __nanosleep(32);
        }
    }
    return true;
}

// The plane block of batch b of a B / C item (16 N complex, contiguous, read only by that batch) is in
// the stage: its L2 lines hold dead data until pair p + R rewrites them -- drop them instead of
// letting the L2 write them back (experiment R6c / R6d, ACP_F2C_DISCARD).
template <int N>
__device__ __forceinline__ void f2c_discard(const F2cArgs& g, const Item& it, int b, int lane, int nl) {
    using K = F2C<N>;
    const size_t NN = (size_t)N * N;
    const char* blk = reinterpret_cast<const char*>(g.S + (size_t)(it.p % g.R) * 2 * NN + (it.phase == 2 ? NN : 0) +
                                                    (size_t)((it.q * K::BPI + b) * 16) * N);
    for (int l = lane; l < 16 * N * (int)sizeof(double2) / 128; l += nl)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(blk + (size_t)l * 128) : "memory");
}

// Thread 0: fetch batch b of item `it` into stage `buf` (its dependencies hold).
template <int N>
__device__ __forceinline__ void issue_batch(const F2cArgs& g, const Item& it, int b, double2* buf,
                                            unsigned long long* bar) {
    using K = F2C<N>;
    const int p = it.p;
    const size_t NN = (size_t)N * N;
    const int base = (it.q * K::BPI + b) * 16;
    const unsigned bytes = 16u * N * sizeof(double2);
    if (it.phase == 0) {
        const FopArgs& a = g.a;
        const int c0 = 2 * p;
        const bool h1 = c0 + 1 < a.n;
        const unsigned half = 16u * N * sizeof(double);
        const unsigned long long pl = pol_last();  // C re-reads x
        mbar_expect(bar, h1 ? bytes : half);
        bulk_g2s(buf, a.X + (size_t)c0 * g.Ng + (size_t)base * N, half, bar, pl);
        if (h1) bulk_g2s(reinterpret_cast<double*>(buf) + 16 * N, a.X + (size_t)(c0 + 1) * g.Ng + (size_t)base * N,
                         half, bar, pl);
    } else {
        const double2* plane = g.S + (size_t)(p % g.R) * 2 * NN + (it.phase == 2 ? NN : 0);
        mbar_expect(bar, bytes);
        bulk_g2s(buf, plane + (size_t)base * N, bytes, bar, pol_first());
    }
}

template <int N>
__device__ __forceinline__ double f2c_symbol(const F2cArgs& g, const double* hk0, const double* hk1, int k0, int k1) {
    const FopArgs& a = g.a;
    if (a.sym < 0) return ld_nc(&a.mult[(size_t)k0 * N + k1]);
    const double h = hk0[k0] + hk1[k1];
    if (a.sym == MULT_KINETIC) return h * g.invN;
    const double d = h + a.tau;  // MULT_PRECOND: 1/(h + tau), rcp estimate + two Newton steps
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = r * (2.0 - d * r);
    r = r * (2.0 - d * r);
    return r * g.invN;
}

// One batch of an item, its input already in `sm` (the stage).  Returns via d[] the partial dots.
template <int N>
__device__ __forceinline__ void f2c_batch(const F2cArgs& g, const Item& it, int b, double2* sm,
                                          const double2* __restrict__ tws, const double* hk0, const double* hk1,
                                          double* d) {
    using namespace f2c;
    using K = F2C<N>;
    constexpr int N2 = K::N2, TB = K::TB, TB2 = K::TB2;
    const FopArgs& a = g.a;
    const int t = threadIdx.x;
    const int p = it.p, c0 = 2 * p, c1 = c0 + 1;
    const bool h1 = c1 < a.n;
    const size_t NN = (size_t)N * N;
    double2* S1 = g.S + (size_t)(p % g.R) * 2 * NN;
    double2* S2 = S1 + NN;
    const int base = (it.q * K::BPI + b) * 16;

    if (it.phase == 0) {
        // ---------------- A: rows base .. base+15 -> S1[k1][i0]
        {
            const int r = t >> 4, n1 = t & 15;
            const double* x0s = reinterpret_cast<const double*>(sm);
            double2 z[N2];
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) {
                const int o = r * N + n1 + 16 * n2;
                z[n2] = mk(x0s[o], h1 ? x0s[16 * N + o] : 0.0);
            }
            dft<N2>(z);
#pragma unroll
            for (int k2 = 1; k2 < N2; ++k2) z[k2] = mul(z[k2], tws[n1 * k2]);
            __syncthreads();  // the stage is read: the exchange overwrites it in place
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) sm[r * TB + k2 * 17 + n1] = z[k2];
        }
        __syncthreads();
        if ((t >> 4) < N2) {
            const int r = t & 15, k2 = t >> 4;
            double2 u[16];
#pragma unroll
            for (int n1 = 0; n1 < 16; ++n1) u[n1] = sm[r * TB + k2 * 17 + n1];
            dft<16>(u);
#pragma unroll
            for (int k1 = 0; k1 < 16; ++k1) __stcg(&S1[(size_t)(N2 * k1 + k2) * N + base + r], u[k1]);
        }
    } else if (it.phase == 1) {
        // ---------------- B: columns base .. base+15: FFT, conj(m .), FFT -> S2[i0][k1]
        {
            const int c = t >> 4, n1 = t & 15;
            double2 z[N2];
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) z[n2] = sm[c * N + n1 + 16 * n2];
            dft<N2>(z);
#pragma unroll
            for (int k2 = 1; k2 < N2; ++k2) z[k2] = mul(z[k2], tws[n1 * k2]);
            __syncthreads();
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) sm[c * TB + k2 * 17 + n1] = z[k2];
        }
        __syncthreads();
        {
            const int c = t >> 4, k2 = t & 15;
            double2 u[16];
            const bool act = k2 < N2;
            if (act) {
#pragma unroll
                for (int n1 = 0; n1 < 16; ++n1) u[n1] = sm[c * TB + k2 * 17 + n1];
                dft<16>(u);  // u[k1] = Zhat[k0 = N2 k1 + k2][base + c]
#pragma unroll
                for (int k1 = 0; k1 < 16; ++k1) {
                    const double m = f2c_symbol<N>(g, hk0, hk1, N2 * k1 + k2, base + c);
                    u[k1] = mk(m * u[k1].x, -m * u[k1].y);
                }
                // second transform, factors swapped: this thread (n1' = k2) holds elements
                // k2 + N2 n2' (n2' = k1 < 16)
                dft<16>(u);
#pragma unroll
                for (int q = 1; q < 16; ++q) u[q] = mul(u[q], tws[k2 * q]);
            }
            __syncthreads();  // every read of the first exchange is done
            if (act) {
#pragma unroll
                for (int q = 0; q < 16; ++q) sm[c * TB2 + q * (N2 + 1) + k2] = u[q];
            }
        }
        __syncthreads();
        {
            const int c = t & 15, q = t >> 4;
            double2 v[N2];
#pragma unroll
            for (int n1 = 0; n1 < N2; ++n1) v[n1] = sm[c * TB2 + q * (N2 + 1) + n1];
            dft<N2>(v);  // v[k1'] = row i0 = 16 k1' + q of column base + c
#pragma unroll
            for (int k1 = 0; k1 < N2; ++k1) __stcg(&S2[(size_t)(16 * k1 + q) * N + base + c], v[k1]);
        }
    } else {
        // ---------------- C: rows base .. base+15 of S2, epilogue
        // the epilogue's x / V values are requested first: their latency hides behind the FFTs
        const int k2 = t & 15, r = t >> 4;
        const bool act2 = k2 < N2;
        const size_t row = (size_t)(base + r) * N;
        const double* x0 = a.X + (size_t)c0 * g.Ng;
        const double* x1 = a.X + (size_t)c1 * g.Ng;
        double e0[16], e1[16], ev[16];
        if (act2) {
            const unsigned long long pf = pol_first();
#pragma unroll
            for (int k1 = 0; k1 < 16; ++k1) {
                const size_t o = row + N2 * k1 + k2;
                e0[k1] = ld_hint(x0 + o, pf);
                e1[k1] = h1 ? ld_hint(x1 + o, pf) : 0.0;
                ev[k1] = a.diag ? ld_nc(a.diag + o) : 0.0;
            }
        }
        {
            const int rr = t >> 4, n1 = t & 15;
            double2 z[N2];
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) z[n2] = sm[rr * N + n1 + 16 * n2];
            dft<N2>(z);
#pragma unroll
            for (int q = 1; q < N2; ++q) z[q] = mul(z[q], tws[n1 * q]);
            __syncthreads();
#pragma unroll
            for (int q = 0; q < N2; ++q) sm[rr * TB + q * 17 + n1] = z[q];
        }
        __syncthreads();
        if (act2) {
            double2 u[16];
#pragma unroll
            for (int n1 = 0; n1 < 16; ++n1) u[n1] = sm[r * TB + k2 * 17 + n1];
            dft<16>(u);
            const unsigned long long pf = pol_first();
            const bool act0 = !a.active || a.active[c0];
            const bool act1 = h1 && (!a.active || a.active[c1]);
            const double s0 = a.shift ? a.shift[c0] : 0.0;
            const double s1 = (a.shift && h1) ? a.shift[c1] : 0.0;
            double* y0 = a.Y + (size_t)c0 * g.Ng;
            double* y1 = a.Y + (size_t)c1 * g.Ng;
#pragma unroll
            for (int k1 = 0; k1 < 16; ++k1) {
                const size_t o = row + N2 * k1 + k2;
                const double u0 = e0[k1], u1 = e1[k1];
                double v0 = u[k1].x, v1 = -u[k1].y;
                if (a.diag) {
                    v0 += (ev[k1] - s0) * u0;
                    v1 += (ev[k1] - s1) * u1;
                } else if (a.shift) {
                    v0 -= s0 * u0;
                    v1 -= s1 * u1;
                }
                if (act0) st_hint(y0 + o, v0, pf);
                if (act1) st_hint(y1 + o, v1, pf);
                d[0] += u0 * v0;
                d[1] += u0 * u0;
                d[2] += u1 * v1;
                d[3] += u1 * u1;
            }
        }
    }
}

// MB = resident CTAs per SM the register budget is sized for (A/B by ACP_F2C_MB).
template <int N, int MB>
__global__ void __launch_bounds__(256, MB) k_f2c(F2cArgs g) {
    using K = F2C<N>;
    extern __shared__ __align__(128) double2 sm[];
    __shared__ __align__(8) unsigned long long bars[2];
    __shared__ double red[8][4];
    __shared__ int s_item;
    __shared__ double2 tws[N];   // exp(-2 pi i j / N): the twiddles of both register passes
    __shared__ double hk[2][N];  // |k_a|^2 / 2 per axis and bin
    const int t = threadIdx.x;
    for (int j = t; j < N; j += blockDim.x) {
        tws[j] = g.tw[j];
        const int m = j < (N + 1) / 2 ? j : j - N;
        hk[0][j] = 0.5 * (m * g.dk0) * (m * g.dk0);
        hk[1][j] = 0.5 * (m * g.dk1) * (m * g.dk1);
    }
    if (t == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    int* cnt = g.queue + 1;
    unsigned uses[2] = {0, 0};  // completed phases of each stage's mbarrier (parity)
    // the item being computed and the next batch to fetch (thread 0 fetches one batch ahead)
    if (t == 0) s_item = atomicAdd(g.queue, 1);
    __syncthreads();
    Item cur = decode<N>(g, s_item);
    int cb = 0, buf = 0;
    if (t == 0 && cur.skip == 0) {
        deps_ready<N>(g, cur, true);  // holds nothing yet: may wait
        issue_batch<N>(g, cur, 0, sm, &bars[0]);
    }
    double d[4] = {0.0, 0.0, 0.0, 0.0};
    while (cur.skip != 3) {
        // ---- the next batch (same item, or batch 0 of the next dequeued item) goes to stage buf^1
        Item nxt = cur;
        int nb = cb + 1;
        const bool last = cur.skip != 0 || nb == K::BPI;
        if (last) {
            __syncthreads();  // everyone has read s_item
            if (t == 0) s_item = atomicAdd(g.queue, 1);
            __syncthreads();
            nxt = decode<N>(g, s_item);
            nb = 0;
        }
        // prefetch only if it cannot block (same item, or producers already done); else after the
        // current item is counted
        bool pre = false;
        if (t == 0 && nxt.skip == 0 && (nb > 0 || deps_ready<N>(g, nxt, false))) {
            issue_batch<N>(g, nxt, nb, sm + (size_t)(buf ^ 1) * K::BUF, &bars[buf ^ 1]);
            pre = true;
        }
        // ---- compute the current batch
        if (cur.skip == 0) {
            mbar_wait(&bars[buf], uses[buf] & 1);
            ++uses[buf];
            if (ACP_F2C_DISCARD == 1 && cur.phase != 0) f2c_discard<N>(g, cur, cb, t, 256);
            f2c_batch<N>(g, cur, cb, sm + (size_t)buf * K::BUF, tws, hk[0], hk[1], d);
            if (ACP_F2C_DISCARD == 2 && cur.phase != 0) f2c_discard<N>(g, cur, cb, t, 256);
            if (ACP_F2C_DISCARD == 3 && cur.phase != 0 && t >= 224) f2c_discard<N>(g, cur, cb, t - 224, 32);
            fence_proxy_async();  // this stage's generic accesses precede its next bulk refill
        }
        if (last && cur.skip != 2) {
            // the item is complete: partial dots, then count it (after the block barrier one
            // thread makes the block's writes visible at GPU scope -- the fence is cumulative)
            if (cur.phase == 2 && g.a.dots && cur.skip == 0) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) d[q] += __shfl_xor_sync(0xffffffffu, d[q], o);
                if ((t & 31) == 0)
#pragma unroll
                    for (int q = 0; q < 4; ++q) red[t >> 5][q] = d[q];
                __syncthreads();
                if (t < 4) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) s += red[w][t];
                    g.part[((size_t)cur.p * K::IPP + cur.q) * 4 + t] = s;
                }
            }
            __syncthreads();
            if (t == 0) {
                // an inactive pair's items do no work but still keep the ring's slot chain: its
                // counts tell pair p + R that the slot is free, so they may only be given after the
                // slot's previous user (pair p - R) is done with it -- counting them at once let
                // pair p + R overwrite S1 / S2 while pair p - R still read them (outer 1 of c4g:
                // PCG iteration counts varied between identical steps, once no convergence)
                if (cur.skip == 1) deps_ready<N>(g, cur, true);
                __threadfence();
                atomicAdd(&cnt[3 * cur.p + cur.phase], 1);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) d[q] = 0.0;
        }
        __syncthreads();  // stage buf is free for its refill two batches from now
        if (t == 0 && nxt.skip == 0 && !pre) {
            deps_ready<N>(g, nxt, true);  // this CTA holds no unfinished item now
            issue_batch<N>(g, nxt, nb, sm + (size_t)(buf ^ 1) * K::BUF, &bars[buf ^ 1]);
        }
        if (last) {
            cur = nxt;
            cb = 0;
        } else {
            cb = nb;
        }
        buf ^= 1;
    }
}

// Grids the fused kernel handles: square, n = 16 N2 with N2 in {2, 4, 8, 12, 16}.
bool f2c_supported(int n0, int n1) {
    if (n0 != n1 || n0 % 16) return false;
    const int q = n0 / 16;
    return q == 2 || q == 4 || q == 8 || q == 12 || q == 16;
}

static int f2c_mb(int N) {
    const char* e = getenv("ACP_F2C_MB");
    if (e) return atoi(e) == 2 ? 2 : 1;
    return 1;
}

template <int N>
static const void* f2c_kernel_n() {
    return f2c_mb(N) == 2 ? (const void*)k_f2c<N, 2> : (const void*)k_f2c<N, 1>;
}

static const void* f2c_kernel(int N) {
    switch (N) {
        case 32: return f2c_kernel_n<32>();
        case 64: return f2c_kernel_n<64>();
        case 128: return f2c_kernel_n<128>();
        case 192: return f2c_kernel_n<192>();
        case 256: return f2c_kernel_n<256>();
        default: ACP_REQUIRE(false, "fused 2D FFT: unsupported grid");
    }
    return nullptr;
}

// Persistent grid (resident CTAs), queue skew d and ring size R for this grid.
struct F2cGeom {
    int grid, d, R;
};

static F2cGeom f2c_geom(acp_context* ctx) {
    const int N = ctx->n[0];
    const void* kern = f2c_kernel(N);
    const size_t smem = f2c_smem(N);
    func_attr(kern, smem);
    if (ctx->f2c_maxcl <= 0) {
        int occ = 0, sms = 0;
        ACP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem));
        ACP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
        ACP_REQUIRE(occ >= 1, "fused 2D FFT: kernel does not fit");
        ctx->f2c_maxcl = occ * sms;
    }
    const int ipp = f2c_ipp(N);
    F2cGeom G;
    G.grid = ctx->f2c_maxcl;
    // the grid holds ~grid items at once (3 ipp per step); B / C items trail by d steps.  What
    // matters is the ring (R = 2d + 4 slots, 2 MB each at 256^2): best at R ~ 36-44 (72-88 MB, L2-
    // resident) -- c4g at 4 batches per item: d = 12 / 16 / 20 / 28 / 36: 27.9 / 25.54 / 25.50 / 26.1 /
    // 27.0 ms; at 2 per item d = 9 / 16 / 32: 27.93 / 26.96 / 27.7 (runs R5b, R5g)
    G.d = (G.grid + 3 * ipp - 1) / (3 * ipp) + 6;
    if (const char* e = getenv("ACP_F2C_SKEW")) G.d = std::max(1, atoi(e));
    G.R = 2 * G.d + 4;
    return G;
}

size_t f2c_scratch_bytes(acp_context* ctx, int n) {
    const int npair = (n + 1) / 2;
    const F2cGeom G = f2c_geom(ctx);
    const size_t NN = (size_t)ctx->n[0] * ctx->n[0];
    return (size_t)std::min(G.R, npair) * 2 * NN * sizeof(double2);
}

size_t f2c_queue_ints(int n) { return 1 + 3 * (size_t)((n + 1) / 2); }
int f2c_items_per_phase(int N) { return f2c_ipp(N); }

void launch_f2c(acp_context* ctx, const FopArgs& a, double2* S, int* queue, double* part, const double2* tw) {
    const int N = ctx->n[0];
    const F2cGeom G = f2c_geom(ctx);
    F2cArgs g;
    g.a = a;
    g.N = N;
    g.Ng = ctx->Ng;
    g.dk0 = 2.0 * M_PI / ctx->sys.cell[0];
    g.dk1 = 2.0 * M_PI / ctx->sys.cell[1];
    g.invN = 1.0 / (double)ctx->Ng;
    g.tw = tw;
    g.S = S;
    g.npair = (a.n + 1) / 2;
    g.R = std::min(G.R, g.npair);
    g.d = G.d;
    g.nsteps = g.npair + 2 * G.d;
    g.queue = queue;
    g.part = part;
    ACP_CUDA(cudaMemsetAsync(queue, 0, f2c_queue_ints(a.n) * sizeof(int), ctx->stream));
    const int grid = std::min(G.grid, g.nsteps * 3 * f2c_ipp(N));
    void* args[] = {&g};
    ACP_CUDA(cudaLaunchKernel(f2c_kernel(N), dim3(grid), dim3(256), args, f2c_smem(N), ctx->stream));
    launched(ctx);
}

}  // namespace acp
