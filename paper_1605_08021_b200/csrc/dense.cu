// dense.cu -- small dense fp64 kernels kept on the device: LU solve (SMW core of
// Eq. dyson4), cyclic Jacobi symmetric eigensolver (phonon modes
// D u = omega^2 u; Rayleigh-Ritz in the ground state) and Cholesky.
// All run in ONE CTA (the matrices are O(N_e) x O(N_e) and off the bandwidth-
// critical loop); reductions use fixed orders, so results are deterministic.
#include "common.cuh"

#include <cmath>

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

// LU with partial pivoting of A (n x n col-major) applied to B (n x nrhs), then back substitution.
// The working copy of A lives in shared memory when it fits (n <= 160), else in place in global
// memory.  Only U is kept (B is eliminated alongside), so each step is: pivot search, row swap,
// rank-1 update with l_ik = A_ik / A_kk formed on the fly -- two barriers per column.
__global__ void __launch_bounds__(1024) k_lu_solve(double* __restrict__ Ag, int n, double* __restrict__ B, int nrhs,
                                                   int use_smem, int* __restrict__ status) {
    extern __shared__ double lsm[];
    __shared__ double sv[32];
    __shared__ int si[32];
    const int tid = threadIdx.x, nt = blockDim.x;
    double* A = Ag;
    if (use_smem) {
        A = lsm;
        for (long long e = tid; e < (long long)n * n; e += nt) A[e] = Ag[e];
        __syncthreads();
    }
    for (int k = 0; k < n; ++k) {
        double bv = -1.0;
        int bi = 1 << 30;
        for (int i = k + tid; i < n; i += nt) {
            const double a = fabs(A[(size_t)k * n + i]);
            if (a > bv) {
                bv = a;
                bi = i;
            }
        }
        double best;
        int p;
        block_argmax_abs(bv, bi, sv, si, best, p);
        if (best == 0.0) {
            if (tid == 0) *status = 1;
            return;
        }
        if (p != k) {
            for (int j = tid; j < n + nrhs; j += nt) {
                double* base = (j < n) ? A + (size_t)j * n : B + (size_t)(j - n) * n;
                const double t = base[k];
                base[k] = base[p];
                base[p] = t;
            }
            __syncthreads();
        }
        const double piv = A[(size_t)k * n + k];
        // rank-1 update: warps over columns (trailing A columns, then B columns), lanes over rows
        const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
        const int ncols = (n - k - 1) + nrhs;
        for (int jj = warp; jj < ncols; jj += nwarp) {
            double* colj = (jj < n - k - 1) ? A + (size_t)(k + 1 + jj) * n : B + (size_t)(jj - (n - k - 1)) * n;
            const double akj = colj[k];
            for (int i = k + 1 + lane; i < n; i += 32) colj[i] -= (A[(size_t)k * n + i] / piv) * akj;
        }
        __syncthreads();
    }
    // back substitution: warps over right-hand sides, lanes over rows
    {
        const int warp = tid >> 5, lane = tid & 31, nwarp = nt >> 5;
        for (int k = n - 1; k >= 0; --k) {
            const double d = A[(size_t)k * n + k];
            for (int j = warp; j < nrhs; j += nwarp) {
                double* bj = B + (size_t)j * n;
                const double x = bj[k] / d;
                __syncwarp();
                if (lane == 0) bj[k] = x;
                for (int i = lane; i < k; i += 32) bj[i] -= A[(size_t)k * n + i] * x;
            }
            __syncthreads();
        }
    }
    if (tid == 0) *status = 0;
}

void lu_solve(acp_context* ctx, double* A, int n, double* B, int nrhs) {
    int* st = ctx->wsi("lu_status", 1);
    const size_t bytes = (size_t)n * n * sizeof(double);
    const int use_smem = bytes <= 200 * 1024;
    static bool attr = false;
    if (!attr) {
        ACP_CUDA(cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    k_lu_solve<<<1, 1024, use_smem ? bytes : 0, ctx->stream>>>(A, n, B, nrhs, use_smem, st);
    launched(ctx);
    int* hp = static_cast<int*>(ctx->pinned);
    ACP_CUDA(cudaMemcpyAsync(hp, st, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    ACP_CUDA(cudaStreamSynchronize(ctx->stream));
    const int h = *hp;
    if (h != 0) throw Error(ACP_ERR_SINGULAR, "singular matrix in LU solve (n = " + std::to_string(n) + ")");
}

// Cyclic (round-robin ordered) Jacobi: A (n x n col-major, symmetric) -> eigenvalues w (ascending),
// eigenvectors V (n x n col-major) if V != nullptr.  Work arrays in global memory.
__global__ void __launch_bounds__(1024) k_jacobi(double* __restrict__ Ag, int n, double* __restrict__ V,
                                                 double* __restrict__ w, int* __restrict__ order,
                                                 double* __restrict__ rot, int max_sweeps, int use_smem) {
    extern __shared__ double jsm[];
    __shared__ double red[32];
    __shared__ int s_done;
    const int tid = threadIdx.x, nt = blockDim.x;
    double* A = Ag;
    if (use_smem) {
        A = jsm;
        for (long long e = tid; e < (long long)n * n; e += nt) A[e] = Ag[e];
        __syncthreads();
    }
    const int m = (n % 2) ? n + 1 : n;  // padded size for the tournament (index n is a dummy)
    if (V)
        for (long long e = tid; e < (long long)n * n; e += nt) V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
    for (int i = tid; i < m; i += nt) order[i] = i;
    __syncthreads();
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        // off-diagonal and total Frobenius norms
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
        if ((tid & 31) == 0) red[tid >> 5] = off;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int i = 0; i < nt / 32; ++i) s += red[i];
            red[0] = s;
        }
        __syncthreads();
        const double offs = red[0];
        __syncthreads();
        if ((tid & 31) == 0) red[tid >> 5] = tot;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int i = 0; i < nt / 32; ++i) s += red[i];
            // converged when the off-diagonal Frobenius norm is below 1e-13 of the total:
            // eigenvalue errors are second order in it (<= 1e-26 relative)
            s_done = (offs <= 1e-26 * s) ? 1 : 0;
        }
        __syncthreads();
        if (s_done) break;
        for (int round = 0; round < m - 1; ++round) {
            const int np = m / 2;
            // rotation for each pair (order[k], order[m-1-k])
            for (int k = tid; k < np; k += nt) {
                int p = order[k], q = order[m - 1 - k];
                if (p > q) {
                    int t = p;
                    p = q;
                    q = t;
                }
                double c = 1.0, s = 0.0;
                if (q < n) {
                    const double apq = A[(size_t)q * n + p];
                    if (apq != 0.0) {
                        const double app = A[(size_t)p * n + p], aqq = A[(size_t)q * n + q];
                        const double th = (aqq - app) / (2.0 * apq);
                        const double t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
                        c = 1.0 / sqrt(t * t + 1.0);
                        s = t * c;
                    }
                }
                rot[4 * k] = c;
                rot[4 * k + 1] = s;
                rot[4 * k + 2] = p;
                rot[4 * k + 3] = q;
            }
            __syncthreads();
            // columns: A <- A J   (warps over pairs, lanes over rows)
            for (int k = tid >> 5; k < np; k += nt >> 5)
                for (int i = tid & 31; i < n; i += 32) {
                const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
                if (q >= n) continue;
                const double c = rot[4 * k], s = rot[4 * k + 1];
                const double aip = A[(size_t)p * n + i], aiq = A[(size_t)q * n + i];
                A[(size_t)p * n + i] = c * aip - s * aiq;
                A[(size_t)q * n + i] = s * aip + c * aiq;
                if (V) {
                    const double vip = V[(size_t)p * n + i], viq = V[(size_t)q * n + i];
                    V[(size_t)p * n + i] = c * vip - s * viq;
                    V[(size_t)q * n + i] = s * vip + c * viq;
                }
            }
            __syncthreads();
            // rows: A <- J^T A
            for (int k = tid >> 5; k < np; k += nt >> 5)
                for (int j = tid & 31; j < n; j += 32) {
                const int p = (int)rot[4 * k + 2], q = (int)rot[4 * k + 3];
                if (q >= n) continue;
                const double c = rot[4 * k], s = rot[4 * k + 1];
                const double apj = A[(size_t)j * n + p], aqj = A[(size_t)j * n + q];
                A[(size_t)j * n + p] = c * apj - s * aqj;
                A[(size_t)j * n + q] = s * apj + c * aqj;
            }
            __syncthreads();
            // round-robin rotation of positions 1..m-1
            if (tid == 0) {
                const int last = order[m - 1];
                for (int i = m - 1; i > 1; --i) order[i] = order[i - 1];
                order[1] = last;
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

void sym_eig(acp_context* ctx, double* A, int n, double* w, double* V) {
    double* Vt = V ? ctx->wsd("eig_Vt", (size_t)n * n) : nullptr;
    int* order = ctx->wsi("eig_order", n + 2);
    double* rot = ctx->wsd("eig_rot", 4 * (size_t)(n / 2 + 2));
    const size_t bytes = (size_t)n * n * sizeof(double);
    const int use_smem = bytes <= 200 * 1024;
    static bool attr = false;
    if (!attr) {
        ACP_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        attr = true;
    }
    k_jacobi<<<1, 1024, use_smem ? bytes : 0, ctx->stream>>>(A, n, Vt, w, order, rot, 40, use_smem);
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
        for (long long e = tid; e < (long long)rows * rows; e += nt) {
            const int i = k + 1 + (int)(e % rows), j = k + 1 + (int)(e / rows);
            if (j <= i) A[(size_t)j * n + i] -= A[(size_t)k * n + i] * A[(size_t)k * n + j];
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
