// fft2c.cuh -- register-resident fp64 DFT blocks for the fused 2D Fourier operator (fft2c.cu).
//
// A length-N transform, N = 16 * N2 (N2 in {2, 4, 8, 12, 16}), is done as two register passes
// with ONE shared-memory exchange (Cooley-Tukey, N = N1 * N2 with N1 = 16):
//   n = n1 + 16 n2,  k = N2 k1 + k2,
//   X[N2 k1 + k2] = sum_n1 W16^(n1 k1) W_N^(n1 k2) sum_n2 x[n1 + 16 n2] W_N2^(n2 k2)
// step 1: thread n1 holds x[n1 + 16 n2] (n2 < N2), DFT-N2, twiddle W_N^(n1 k2);
// step 2: thread k2 holds the step-1 outputs of all n1, DFT-16 -> X[N2 k1 + k2] (k1 < 16).
// The same algebra with the factors swapped (N1' = N2, N2' = 16) maps "thread j holds the
// elements j + N2 m" -- exactly what step 2 leaves in thread k2 -- to a second transform, so
// a forward transform followed by an inverse one needs no exchange in between.
//
// Everything here is __host__ __device__ so tools/fft2c_host_test.cu checks it on the CPU.
#pragma once

#include <vector_types.h>

namespace acp {
namespace f2c {

#define F2C_HD __host__ __device__ __forceinline__

F2C_HD double2 mk(double x, double y) {
    double2 r;
    r.x = x;
    r.y = y;
    return r;
}
F2C_HD double2 add(double2 a, double2 b) { return mk(a.x + b.x, a.y + b.y); }
F2C_HD double2 sub(double2 a, double2 b) { return mk(a.x - b.x, a.y - b.y); }
F2C_HD double2 mul(double2 a, double2 b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
F2C_HD double2 mi(double2 a) { return mk(a.y, -a.x); }  // * (-i)

// In-place forward DFT of R values: y_s = sum_r x_r exp(-2 pi i r s / R).
template <int R> F2C_HD void dft(double2* x);

template <> F2C_HD void dft<1>(double2*) {}

template <> F2C_HD void dft<2>(double2* x) {
    const double2 a = x[0], b = x[1];
    x[0] = add(a, b);
    x[1] = sub(a, b);
}

template <> F2C_HD void dft<3>(double2* x) {
    const double s1 = 0.86602540378443864676;  // sin(2 pi / 3)
    const double2 a = add(x[1], x[2]);
    const double2 b = sub(x[1], x[2]);
    const double2 t = mk(x[0].x - 0.5 * a.x, x[0].y - 0.5 * a.y);
    const double2 u = mk(s1 * b.y, -s1 * b.x);  // -i sin(2pi/3) b
    x[0] = add(x[0], a);
    x[1] = add(t, u);
    x[2] = sub(t, u);
}

template <> F2C_HD void dft<4>(double2* x) {
    const double2 t0 = add(x[0], x[2]), t1 = sub(x[0], x[2]);
    const double2 t2 = add(x[1], x[3]), t3 = mi(sub(x[1], x[3]));
    x[0] = add(t0, t2);
    x[2] = sub(t0, t2);
    x[1] = add(t1, t3);
    x[3] = sub(t1, t3);
}

template <> F2C_HD void dft<8>(double2* x) {
    double2 e[4] = {x[0], x[2], x[4], x[6]};
    double2 o[4] = {x[1], x[3], x[5], x[7]};
    dft<4>(e);
    dft<4>(o);
    const double h = 0.70710678118654752440;  // sqrt(1/2)
    const double2 o1 = mk(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));   // W8^1
    const double2 o2 = mi(o[2]);                                            // W8^2
    const double2 o3 = mk(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));  // W8^3
    x[0] = add(e[0], o[0]);
    x[4] = sub(e[0], o[0]);
    x[1] = add(e[1], o1);
    x[5] = sub(e[1], o1);
    x[2] = add(e[2], o2);
    x[6] = sub(e[2], o2);
    x[3] = add(e[3], o3);
    x[7] = sub(e[3], o3);
}

// Radix-4 butterfly on x[i], x[i + s], x[i + 2s], x[i + 3s] in place (compile-time indices, so
// the "in place" is register renaming).
template <int I, int S>
F2C_HD void dft4_at(double2* x) {
    const double2 t0 = add(x[I], x[I + 2 * S]), t1 = sub(x[I], x[I + 2 * S]);
    const double2 t2 = add(x[I + S], x[I + 3 * S]), t3 = mi(sub(x[I + S], x[I + 3 * S]));
    x[I] = add(t0, t2);
    x[I + 2 * S] = sub(t0, t2);
    x[I + S] = add(t1, t3);
    x[I + 3 * S] = sub(t1, t3);
}
template <int I, int S>
F2C_HD void dft3_at(double2* x) {
    const double s1 = 0.86602540378443864676;
    const double2 a = add(x[I + S], x[I + 2 * S]);
    const double2 b = sub(x[I + S], x[I + 2 * S]);
    const double2 t = mk(x[I].x - 0.5 * a.x, x[I].y - 0.5 * a.y);
    const double2 u = mk(s1 * b.y, -s1 * b.x);
    x[I] = add(x[I], a);
    x[I + S] = add(t, u);
    x[I + 2 * S] = sub(t, u);
}
template <int A, int B>
F2C_HD void swp(double2* x) {
    const double2 t = x[A];
    x[A] = x[B];
    x[B] = t;
}

// 12 = 4 x 3, coprime: Good-Thomas (no internal twiddles).  Input n = (3 n1 + 4 n2) mod 12,
// output k = (9 k1 + 4 k2) mod 12 (CRT), X[k] = sum W4^(n1 k1) W3^(n2 k2) x[n].
template <> F2C_HD void dft<12>(double2* x) {
    // gather into a[n2 * 4 + n1] = x[(3 n1 + 4 n2) mod 12] (a permutation: register renaming)
    double2 a[12];
#pragma unroll
    for (int n2 = 0; n2 < 3; ++n2)
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) a[n2 * 4 + n1] = x[(3 * n1 + 4 * n2) % 12];
    dft4_at<0, 1>(a);
    dft4_at<4, 1>(a);
    dft4_at<8, 1>(a);
    dft3_at<0, 4>(a);
    dft3_at<1, 4>(a);
    dft3_at<2, 4>(a);
    dft3_at<3, 4>(a);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1)
#pragma unroll
        for (int k2 = 0; k2 < 3; ++k2) x[(9 * k1 + 4 * k2) % 12] = a[k2 * 4 + k1];
}

// 16 = 4 x 4 with the W16 twiddles between the radix-4 passes:
// X[4 k1 + k2] = sum_n1 W4^(n1 k1) W16^(n1 k2) sum_n2 x[n1 + 4 n2] W4^(n2 k2).
template <> F2C_HD void dft<16>(double2* x) {
    const double c1 = 0.92387953251128675613;  // cos(pi/8)
    const double s1 = 0.38268343236508977173;  // sin(pi/8)
    const double h = 0.70710678118654752440;
    // stage 1: x[n1 + 4 k2] <- A[n1][k2]
    dft4_at<0, 4>(x);
    dft4_at<1, 4>(x);
    dft4_at<2, 4>(x);
    dft4_at<3, 4>(x);
    // W16^(n1 k2) on x[n1 + 4 k2]: W16^1 = (c1, -s1), W16^2 = (h, -h), W16^3 = (s1, -c1),
    // W16^4 = -i, W16^6 = (-h, -h), W16^9 = (-c1, s1)
    x[5] = mul(x[5], mk(c1, -s1));
    x[9] = mk(h * (x[9].x + x[9].y), h * (x[9].y - x[9].x));
    x[13] = mul(x[13], mk(s1, -c1));
    x[6] = mk(h * (x[6].x + x[6].y), h * (x[6].y - x[6].x));
    x[10] = mi(x[10]);
    x[14] = mk(h * (x[14].y - x[14].x), -h * (x[14].x + x[14].y));
    x[7] = mul(x[7], mk(s1, -c1));
    x[11] = mk(h * (x[11].y - x[11].x), -h * (x[11].x + x[11].y));
    x[15] = mul(x[15], mk(-c1, s1));
    // stage 2 over n1 for each k2: x[k1 + 4 k2] <- X[4 k1 + k2]
    dft4_at<0, 1>(x);
    dft4_at<4, 1>(x);
    dft4_at<8, 1>(x);
    dft4_at<12, 1>(x);
    // transpose the 4 x 4 index (k1 + 4 k2 -> 4 k1 + k2)
    swp<1, 4>(x);
    swp<2, 8>(x);
    swp<3, 12>(x);
    swp<6, 9>(x);
    swp<7, 13>(x);
    swp<11, 14>(x);
}

#undef F2C_HD

}  // namespace f2c
}  // namespace acp
