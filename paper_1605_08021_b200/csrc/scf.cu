// scf.cu -- ground state (acp_ground_state): PAPER.md:186-207 (Eqs. Hamil, effV), model
// PAPER.md:822-832; the paper solves it with LOBPCG + Anderson mixing.
//
// B200 design: the eigen-subproblem at every SCF step is solved by Chebyshev-filtered
// subspace iteration (ChFSI) on the block X (N_g x nb), built only from the K1
// Fourier-operator kernel (H apply), the DMMA Gram GEMMs (K2), a device Cholesky and
// a device Jacobi Rayleigh-Ritz.  Density mixing: Anderson acceleration of the
// Kerker-preconditioned residual (same scheme as the oracle; it only changes the
// path to the fixed point).
#include "gemm.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

namespace acp {

// rho(a) = f sum_i Psi(a,i)^2
__global__ void k_density(int Ng, int n_occ, double f, const double* __restrict__ Psi, double* __restrict__ rho) {
    int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= Ng) return;
    double s = 0.0;
    for (int i = 0; i < n_occ; ++i) {
        const double p = Psi[(size_t)i * Ng + a];
        s += p * p;
    }
    rho[a] = f * s;
}

__global__ void k_sum_parts(size_t n, const double* __restrict__ x, const double* __restrict__ y, int mode,
                            double* __restrict__ part) {
    // mode 0: sum x ; mode 1: sum x*x ; mode 2: sum (x-y)^2 ; mode 3: max x
    __shared__ double red[32];
    double s = (mode == 3) ? -1e308 : 0.0;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const double v = x[i];
        if (mode == 0) s += v;
        else if (mode == 1) s += v * v;
        else if (mode == 2) {
            const double d = v - y[i];
            s += d * d;
        } else s = fmax(s, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        double t = __shfl_xor_sync(0xffffffffu, s, o);
        s = (mode == 3) ? fmax(s, t) : s + t;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = (mode == 3) ? -1e308 : 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = (mode == 3) ? fmax(t, red[w]) : t + red[w];
        part[blockIdx.x] = t;
    }
}

static double reduce(acp_context* ctx, const double* x, const double* y, size_t n, int mode) {
    const int blocks = 128;
    double* part = ctx->wsd("scf_part", blocks);
    k_sum_parts<<<blocks, 256, 0, ctx->stream>>>(n, x, y, mode, part);
    launched(ctx);
    double h[blocks];
    ACP_CUDA(cudaMemcpyAsync(h, part, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    double s = (mode == 3) ? -1e308 : 0.0;
    for (int i = 0; i < blocks; ++i) s = (mode == 3) ? std::max(s, h[i]) : s + h[i];
    return s;
}

__global__ void k_axpby(size_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = a * x[i] + (b == 0.0 ? 0.0 : b * y[i]);
}
static void axpby(acp_context* ctx, size_t n, double a, const double* x, double b, double* y) {
    k_axpby<<<cdiv(n, 256), 256, 0, ctx->stream>>>(n, a, x, b, y);
    launched(ctx);
}

// Chebyshev three-term step: Ynew = s1 * HY + s2 * Xold (HY = (H - c) Y precomputed)
__global__ void k_cheb_step(size_t n, double s1, const double* __restrict__ HY, double s2,
                            const double* __restrict__ Xold, double* __restrict__ Ynew) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) Ynew[i] = s1 * HY[i] + s2 * Xold[i];
}

__global__ void k_clip_neg(int n, const double* __restrict__ m, double* __restrict__ rho) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rho[i] = fmax(-m[i], 0.0);
}

__global__ void k_scale(size_t n, double s, double* __restrict__ x) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) x[i] *= s;
}

// Plane-wave start: column j = cos / sin (k_j . r) for the host-sorted list of the lowest
// wave vectors (mode[j] = (m0, m1, kind), kind 0 = constant, 1 = cos, 2 = sin); the first
// Rayleigh-Ritz orthonormalises the block.
__global__ void k_plane_waves(int n0, int n1, int nb, const int* __restrict__ mode, double* __restrict__ X) {
    const size_t Ng = (size_t)n0 * n1;
    size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= Ng * nb) return;
    const int a = (int)(e % Ng), j = (int)(e / Ng);
    const int i0 = a / n1, i1 = a % n1;
    const int m0 = mode[3 * j], m1 = mode[3 * j + 1], kind = mode[3 * j + 2];
    double t = (double)m0 * i0 / n0 + (double)m1 * i1 / n1;
    t -= rint(t);
    double v = 1.0;
    if (kind == 1) v = cospi(2.0 * t);
    else if (kind == 2) v = sinpi(2.0 * t);
    X[e] = v;
}

// Linv (n x n) = L^{-1} for lower-triangular L (col-major), single CTA, column-parallel.
__global__ void k_tri_inv_lower(int n, const double* __restrict__ L, double* __restrict__ Linv) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        // solve L x = e_j  (x_i = 0 for i < j)
        for (int i = 0; i < n; ++i) {
            double v;
            if (i < j) v = 0.0;
            else {
                double s = (i == j) ? 1.0 : 0.0;
                for (int k = j; k < i; ++k) s -= L[(size_t)k * n + i] * Linv[(size_t)j * n + k];
                v = s / L[(size_t)i * n + i];
            }
            Linv[(size_t)j * n + i] = v;
        }
    }
}

__global__ void k_symmetrize(int n, double* __restrict__ A) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    int i = e % n, j = e / n;
    if (i < j) {
        const double v = 0.5 * (A[(size_t)j * n + i] + A[(size_t)i * n + j]);
        A[(size_t)j * n + i] = v;
        A[(size_t)i * n + j] = v;
    }
}

__global__ void k_transpose(int n, const double* __restrict__ A, double* __restrict__ At) {
    int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n * n) return;
    int i = e % n, j = e / n;
    At[(size_t)i * n + j] = A[e];
}

// per-column residual norms^2 of R = HX - X diag(w)
__global__ void k_resid(int Ng, int nb, const double* __restrict__ HX, const double* __restrict__ X,
                        const double* __restrict__ w, double* __restrict__ res) {
    __shared__ double red[32];
    const int j = blockIdx.x;
    double s = 0.0;
    for (int a = threadIdx.x; a < Ng; a += blockDim.x) {
        const double r = HX[(size_t)j * Ng + a] - w[j] * X[(size_t)j * Ng + a];
        s += r * r;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
        res[j] = t;
    }
}

struct Eig {
    acp_context* ctx;
    int Ng, nb;
    double* X;   // Ng x nb (orthonormal, dV-weighted)
    double* Y;
    double* Z;
    double* T;
    double* HX;
    double* S;
    double* Hs;
    double* Linv;
    double* LinvT;
    double* C;
    double* Q;
    double* B;
    double* w;
    double* res;
    const double* multH;
    std::vector<double> hw, hres;

    // Rayleigh-Ritz on span(Y): X <- Y B, HX <- (H Y) B, w <- Ritz values.
    void rayleigh_ritz(const double* V, double* Yin) {
        const double dV = ctx->dV;
        FopArgs f;
        f.X = Yin;
        f.Y = T;
        f.n = nb;
        f.mult = multH;
        f.diag = V;
        fourier_op(ctx, f);
        gemm_tn(ctx, Ng, nb, nb, dV, Yin, Ng, Yin, Ng, S);
        gemm_tn(ctx, Ng, nb, nb, dV, Yin, Ng, T, Ng, Hs);
        cholesky(ctx, S, nb);
        k_tri_inv_lower<<<1, 256, 0, ctx->stream>>>(nb, S, Linv);
        launched(ctx);
        k_transpose<<<cdiv(nb * nb, 256), 256, 0, ctx->stream>>>(nb, Linv, LinvT);
        launched(ctx);
        // C = Linv Hs LinvT
        gemm_nn(ctx, nb, nb, nb, 1.0, Linv, nb, Hs, nb, 0.0, Q, nb);
        gemm_nn(ctx, nb, nb, nb, 1.0, Q, nb, LinvT, nb, 0.0, C, nb);
        k_symmetrize<<<cdiv(nb * nb, 256), 256, 0, ctx->stream>>>(nb, C);
        launched(ctx);
        sym_eig(ctx, C, nb, w, Q);
        gemm_nn(ctx, nb, nb, nb, 1.0, LinvT, nb, Q, nb, 0.0, B, nb);
        gemm_nn(ctx, Ng, nb, nb, 1.0, Yin, Ng, B, nb, 0.0, X, Ng);
        gemm_nn(ctx, Ng, nb, nb, 1.0, T, Ng, B, nb, 0.0, HX, Ng);
        k_resid<<<nb, 256, 0, ctx->stream>>>(Ng, nb, HX, X, w, res);
        launched(ctx);
        ACP_CUDA(cudaMemcpyAsync(hw.data(), w, nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        ACP_CUDA(cudaMemcpyAsync(hres.data(), res, nb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    }

    // Y = p_m(H) X, Chebyshev filter damping [a, b] (scaled recurrence, Zhou & Saad).
    void filter(const double* V, int m, double a, double b, double a0) {
        const size_t tot = (size_t)Ng * nb;
        const double e = 0.5 * (b - a), c = 0.5 * (b + a);
        double sigma = e / (a0 - c);
        const double sigma1 = sigma;
        double* shift = ctx->wsd("eig_shift", nb);
        fill(ctx, shift, nb, c);
        FopArgs f;
        f.n = nb;
        f.mult = multH;
        f.diag = V;
        f.shift = shift;
        // Y = (H - c) X * sigma1 / e
        f.X = X;
        f.Y = T;
        fourier_op(ctx, f);
        axpby(ctx, tot, sigma1 / e, T, 0.0, Y);
        double* Xo = X;  // previous
        double* Yc = Y;  // current
        double* Yn = Z;  // next
        // keep X intact: copy into the rotation buffers
        copy_cols(ctx, HX, X, tot);  // HX used as "previous" storage during filtering
        Xo = HX;
        for (int i = 2; i <= m; ++i) {
            const double sigma2 = 1.0 / (2.0 / sigma1 - sigma);
            f.X = Yc;
            f.Y = T;
            fourier_op(ctx, f);
            k_cheb_step<<<cdiv(tot, 256), 256, 0, ctx->stream>>>(tot, 2.0 * sigma2 / e, T, -sigma * sigma2, Xo, Yn);
            launched(ctx);
            double* t = Xo;
            Xo = Yc;
            Yc = Yn;
            Yn = t;
            sigma = sigma2;
        }
        if (Yc != Y) copy_cols(ctx, Y, Yc, tot);
    }
};

void ground_state(acp_context* ctx, const double* h_R, const acp_scf_opts& o, double* Psi, double* eps, double* rho,
                  double* V, double* G, double* h_info) {
    const int Ng = ctx->Ng;
    const int NA = ctx->sys.n_atoms;
    const int n_occ = ctx->sys.n_occ;
    const int nb = n_occ + std::max(1, o.n_extra);
    ACP_REQUIRE(nb < Ng, "too many eigenpairs for the grid");
    ACP_REQUIRE(nb <= 1024, "block too large");
    const double Ne = ctx->sys.Z * NA;
    const size_t tot = (size_t)Ng * nb;
    const int dim = ctx->dim;
    double* dR = ctx->wsd("gs_R", (size_t)NA * dim);
    ACP_CUDA(cudaMemcpyAsync(dR, h_R, (size_t)NA * dim * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    if (G) perturbations(ctx, h_R, G);
    // pseudocharge m
    double2* spec = static_cast<double2*>(ctx->ws("gs_spec", (size_t)Ng * sizeof(double2)));
    spectrum_m(ctx, dR, spec);
    double* m = ctx->wsd("gs_m", Ng);
    ifft_hermitian(ctx, spec, 1, m);
    // initial density: clip(-m) scaled to Ne
    double* rin = ctx->wsd("gs_rin", Ng);
    k_clip_neg<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(Ng, m, rin);
    launched(ctx);
    {
        const double s = reduce(ctx, rin, nullptr, Ng, 0) * ctx->dV;
        k_scale<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(Ng, Ne / s, rin);
        launched(ctx);
    }
    // multipliers
    double* multH = ctx->wsd("gs_multH", Ng);
    copy_cols(ctx, multH, multiplier(ctx, MULT_KINETIC, 0.0), Ng);
    double* multK = ctx->wsd("gs_multK", Ng);
    copy_cols(ctx, multK, multiplier(ctx, MULT_YUKAWA, 0.0), Ng);
    double* multKer = ctx->wsd("gs_multKer", Ng);
    {
        std::vector<double> k2(Ng), mk(Ng);
        ACP_CUDA(cudaMemcpy(k2.data(), ctx->d_k2, Ng * sizeof(double), cudaMemcpyDeviceToHost));
        for (int i = 0; i < Ng; ++i)
            mk[i] = (i == 0) ? 0.0 : k2[i] / (k2[i] + o.kerker_k0 * o.kerker_k0) / (double)Ng;
        ACP_CUDA(cudaMemcpy(multKer, mk.data(), Ng * sizeof(double), cudaMemcpyHostToDevice));
    }
    double kmax2 = 0.0;
    {
        std::vector<double> k2(Ng);
        ACP_CUDA(cudaMemcpy(k2.data(), ctx->d_k2, Ng * sizeof(double), cudaMemcpyDeviceToHost));
        for (double v : k2) kmax2 = std::max(kmax2, v);
    }
    Eig E;
    E.ctx = ctx;
    E.Ng = Ng;
    E.nb = nb;
    E.X = ctx->wsd("gs_X", tot);
    E.Y = ctx->wsd("gs_Y", tot);
    E.Z = ctx->wsd("gs_Z", tot);
    E.T = ctx->wsd("gs_T", tot);
    E.HX = ctx->wsd("gs_HX", tot);
    E.S = ctx->wsd("gs_S", (size_t)nb * nb);
    E.Hs = ctx->wsd("gs_Hs", (size_t)nb * nb);
    E.Linv = ctx->wsd("gs_Linv", (size_t)nb * nb);
    E.LinvT = ctx->wsd("gs_LinvT", (size_t)nb * nb);
    E.C = ctx->wsd("gs_C", (size_t)nb * nb);
    E.Q = ctx->wsd("gs_Q", (size_t)nb * nb);
    E.B = ctx->wsd("gs_B", (size_t)nb * nb);
    E.w = ctx->wsd("gs_w", nb);
    E.res = ctx->wsd("gs_res", nb);
    E.multH = multH;
    E.hw.resize(nb);
    E.hres.resize(nb);
    {
        // lowest |k|^2 wave vectors on a half plane (m0 > 0, or m0 == 0 and m1 > 0), cos and sin each
        const int n0 = ctx->n[0], n1 = ctx->n[1];
        const double L0 = ctx->sys.cell[0], L1 = dim == 2 ? ctx->sys.cell[1] : 1.0;
        std::vector<std::pair<double, std::pair<int, int>>> ks;
        // enough wave vectors for nb functions (1D: nb/2 + 1; 2D: a disc of radius ~sqrt(nb))
        const int rr = (int)std::sqrt((double)nb) + 4;
        const int r0 = dim == 2 ? std::min(n0 / 2 - 1, rr) : std::min(n0 / 2 - 1, nb / 2 + 2);
        const int r1 = dim == 2 ? std::min(n1 / 2 - 1, rr) : 0;
        for (int m0 = 0; m0 <= r0; ++m0)
            for (int m1 = -r1; m1 <= r1; ++m1) {
                if (m0 == 0 && m1 <= 0) continue;
                const double k2v = (m0 / L0) * (m0 / L0) + (dim == 2 ? (m1 / L1) * (m1 / L1) : 0.0);
                ks.push_back({k2v, {m0, m1}});
            }
        std::stable_sort(ks.begin(), ks.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
        std::vector<int> mode(3 * (size_t)nb);
        mode[0] = mode[1] = mode[2] = 0;
        for (int j = 1; j < nb; ++j) {
            const auto& kk = ks.at((size_t)(j - 1) / 2).second;
            mode[3 * j] = kk.first;
            mode[3 * j + 1] = kk.second;
            mode[3 * j + 2] = (j % 2) ? 1 : 2;
        }
        int* dmode = ctx->wsi("gs_mode", 3 * (size_t)nb);
        ACP_CUDA(cudaMemcpy(dmode, mode.data(), mode.size() * sizeof(int), cudaMemcpyHostToDevice));
        k_plane_waves<<<cdiv(tot, 256), 256, 0, ctx->stream>>>(n0, n1, nb, dmode, E.X);
        launched(ctx);
    }
    // Anderson history
    const int hist = std::max(1, o.history);
    double* Xh = ctx->wsd("gs_Xh", (size_t)Ng * (hist + 1));
    double* Fh = ctx->wsd("gs_Fh", (size_t)Ng * (hist + 1));
    double* dX = ctx->wsd("gs_dX", (size_t)Ng * hist);
    double* dF = ctx->wsd("gs_dF", (size_t)Ng * hist);
    double* Gm = ctx->wsd("gs_Gm", (size_t)hist * hist);
    double* gv = ctx->wsd("gs_gv", hist);
    double* fres = ctx->wsd("gs_f", Ng);
    double* rout = ctx->wsd("gs_rout", Ng);
    double* diff = ctx->wsd("gs_diff", Ng);
    const bool debug = getenv("ACP_DEBUG") != nullptr;
    long passes_total = 0;
    std::vector<int> order;  // history slots, oldest first (ring of hist+1 slots)
    double err = 1e300;
    int it = 0;
    for (it = 1; it <= o.max_scf_iter; ++it) {
        // V = K * (rho + m)
        axpby(ctx, Ng, 1.0, rin, 0.0, diff);
        axpby(ctx, Ng, 1.0, m, 1.0, diff);
        FopArgs fk;
        fk.X = diff;
        fk.Y = V;
        fk.n = 1;
        fk.mult = multK;
        fourier_op(ctx, fk);
        const double vmax = reduce(ctx, V, nullptr, Ng, 3);
        const double b = 0.5 * kmax2 + vmax + 1.0;
        // eigen-solve to a tolerance that tightens with the SCF residual
        const double etol = std::max(o.eig_tol, std::min(1e-4, 1e-2 * err));
        copy_cols(ctx, E.Y, E.X, tot);
        E.rayleigh_ritz(V, E.Y);
        double rprev = 1e300;
        for (int pass = 0; pass < 400; ++pass) {
            double rmax = 0.0;
            for (int j = 0; j < n_occ; ++j) rmax = std::max(rmax, std::sqrt(E.hres[j] * ctx->dV));
            if (rmax <= etol) break;
            if (rmax > 0.9 * rprev && rmax < 1e-11) break;  // rounding floor reached
            rprev = rmax;
            const double a = E.hw[nb - 1];
            const double a0 = E.hw[0];
            E.filter(V, 40, a, b, a0);
            ++passes_total;
            E.rayleigh_ritz(V, E.Y);
        }
        // rho_out
        k_density<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(Ng, n_occ, ctx->sys.occ, E.X, rout);
        launched(ctx);
        err = std::sqrt(reduce(ctx, rout, rin, Ng, 2) / reduce(ctx, rin, nullptr, Ng, 1));
        if (debug) {
            double rmax = 0.0;
            for (int j = 0; j <= n_occ && j < nb; ++j) rmax = std::max(rmax, std::sqrt(E.hres[j] * ctx->dV));
            fprintf(stderr, "[acp scf] it %4d  res %.3e  eig-res(occ+lumo) %.2e  passes %ld  gap %.6f\n", it, err, rmax,
                    passes_total, E.hw[n_occ] - E.hw[n_occ - 1]);
        }
        if (err <= o.scf_tol) break;
        // f = Kerker(rho_out - rho_in)
        axpby(ctx, Ng, 1.0, rout, 0.0, diff);
        axpby(ctx, Ng, -1.0, rin, 1.0, diff);
        FopArgs fp;
        fp.X = diff;
        fp.Y = fres;
        fp.n = 1;
        fp.mult = multKer;
        fourier_op(ctx, fp);
        // push (rin, f) into the history ring (slot order kept on the host; no overlapping copies)
        int slot;
        if ((int)order.size() == hist + 1) {
            slot = order.front();
            order.erase(order.begin());
        } else {
            slot = (int)order.size();
        }
        order.push_back(slot);
        copy_cols(ctx, Xh + (size_t)slot * Ng, rin, Ng);
        copy_cols(ctx, Fh + (size_t)slot * Ng, fres, Ng);
        const int nh = (int)order.size();
        if (nh >= 2) {
            const int k = nh - 1;
            for (int i = 0; i < k; ++i) {
                const double* x1 = Xh + (size_t)order[i + 1] * Ng;
                const double* x0 = Xh + (size_t)order[i] * Ng;
                const double* f1 = Fh + (size_t)order[i + 1] * Ng;
                const double* f0 = Fh + (size_t)order[i] * Ng;
                axpby(ctx, Ng, 1.0, x1, 0.0, dX + (size_t)i * Ng);
                axpby(ctx, Ng, -1.0, x0, 1.0, dX + (size_t)i * Ng);
                axpby(ctx, Ng, 1.0, f1, 0.0, dF + (size_t)i * Ng);
                axpby(ctx, Ng, -1.0, f0, 1.0, dF + (size_t)i * Ng);
            }
            // least squares min ||f - dF gamma|| via the normal equations, regularised
            gemm_tn(ctx, Ng, k, k, 1.0, dF, Ng, dF, Ng, Gm);
            gemm_tn(ctx, Ng, k, 1, 1.0, dF, Ng, fres, Ng, gv);
            std::vector<double> hG((size_t)k * k);
            ACP_CUDA(cudaMemcpyAsync(hG.data(), Gm, hG.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
            ACP_CUDA(cudaStreamSynchronize(ctx->stream));
            double tr = 0.0;
            for (int i = 0; i < k; ++i) tr += hG[(size_t)i * k + i];
            for (int i = 0; i < k; ++i) hG[(size_t)i * k + i] += 1e-13 * tr;
            ACP_CUDA(cudaMemcpyAsync(Gm, hG.data(), hG.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            lu_solve(ctx, Gm, k, gv, 1);
            // rin <- rin + beta f - (dX + beta dF) gamma
            axpby(ctx, Ng, o.beta, fres, 1.0, rin);
            gemm_nn(ctx, Ng, k, 1, -1.0, dX, Ng, gv, k, 1.0, rin, Ng);
            gemm_nn(ctx, Ng, k, 1, -o.beta, dF, Ng, gv, k, 1.0, rin, Ng);
        } else {
            axpby(ctx, Ng, o.beta, fres, 1.0, rin);
        }
        const double s = reduce(ctx, rin, nullptr, Ng, 0) * ctx->dV;
        k_scale<<<cdiv(Ng, 256), 256, 0, ctx->stream>>>(Ng, Ne / s, rin);
        launched(ctx);
    }
    if (err > o.scf_tol)
    {
        char buf[160];
        snprintf(buf, sizeof(buf), "SCF residual %.3e after %d iterations (tol %.1e)", err, o.max_scf_iter, o.scf_tol);
        throw Error(ACP_ERR_NOT_CONVERGED, buf);
    }
    copy_cols(ctx, Psi, E.X, (size_t)Ng * n_occ);
    copy_cols(ctx, eps, E.w, nb);
    copy_cols(ctx, rho, rout, Ng);
    sync(ctx);
    if (h_info) {
        h_info[0] = it;
        h_info[1] = err;
        h_info[2] = E.hw[n_occ] - E.hw[n_occ - 1];
    }
}

}  // namespace acp
