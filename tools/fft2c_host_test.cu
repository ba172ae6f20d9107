// Host check of the register DFT blocks of csrc/fft2c.cuh and of the two-step (16 x N2) scheme
// used by the fused 2D operator, against a naive DFT:  nvcc -x cu -o /tmp/t tools/fft2c_host_test.cu
#include <cmath>
#include <complex>
#include <cstdio>
#include <vector>
#include "../paper_1605_08021_b200/csrc/fft2c.cuh"
using namespace acp::f2c;
typedef std::complex<double> C;

static std::vector<C> naive(const std::vector<C>& x) {
    const int N = x.size();
    std::vector<C> y(N);
    for (int k = 0; k < N; ++k) {
        C s = 0;
        for (int n = 0; n < N; ++n) s += x[n] * std::polar(1.0, -2 * M_PI * (double)((long)n * k % N) / N);
        y[k] = s;
    }
    return y;
}
static double2 d2(C c) { return mk(c.real(), c.imag()); }
static C cc(double2 d) { return C(d.x, d.y); }

template <int R>
static double test_block() {
    std::vector<C> x(R);
    for (int i = 0; i < R; ++i) x[i] = C(std::sin(1.3 * i + 0.2), std::cos(0.7 * i * i + 1));
    double2 r[R];
    for (int i = 0; i < R; ++i) r[i] = d2(x[i]);
    dft<R>(r);
    auto y = naive(x);
    double e = 0;
    for (int i = 0; i < R; ++i) e = std::max(e, std::abs(cc(r[i]) - y[i]));
    return e;
}

// the fused kernel's composition with N1 = 16 threads in step 1 and N2 in step 2 (forward), then
// the swapped factorisation for a second transform straight from the registers of step 2
template <int N2>
static double test_two_step() {
    constexpr int N = 16 * N2;
    std::vector<C> x(N);
    for (int i = 0; i < N; ++i) x[i] = C(std::sin(0.37 * i), std::cos(0.11 * i * i));
    std::vector<double2> tw(N);
    for (int j = 0; j < N; ++j) tw[j] = mk(std::cos(2 * M_PI * j / N), -std::sin(2 * M_PI * j / N));
    double2 T[16][N2];
    for (int n1 = 0; n1 < 16; ++n1) {  // step 1
        double2 z[N2];
        for (int n2 = 0; n2 < N2; ++n2) z[n2] = d2(x[n1 + 16 * n2]);
        dft<N2>(z);
        for (int k2 = 0; k2 < N2; ++k2) T[n1][k2] = mul(z[k2], tw[n1 * k2]);
    }
    double2 R[N2][16];  // thread k2 holds X[N2 k1 + k2] in R[k2][k1]
    for (int k2 = 0; k2 < N2; ++k2) {
        double2 u[16];
        for (int n1 = 0; n1 < 16; ++n1) u[n1] = T[n1][k2];
        dft<16>(u);
        for (int k1 = 0; k1 < 16; ++k1) R[k2][k1] = u[k1];
    }
    auto y = naive(x);
    double e = 0;
    for (int k2 = 0; k2 < N2; ++k2)
        for (int k1 = 0; k1 < 16; ++k1) e = std::max(e, std::abs(cc(R[k2][k1]) - y[N2 * k1 + k2]));
    // second transform (of X itself) with N1' = N2, N2' = 16: thread n1' = k2 holds X[n1' + N2 m]
    double2 T2[N2][16];
    for (int n1 = 0; n1 < N2; ++n1) {
        double2 z[16];
        for (int m = 0; m < 16; ++m) z[m] = R[n1][m];
        dft<16>(z);
        for (int k2 = 0; k2 < 16; ++k2) T2[n1][k2] = mul(z[k2], tw[n1 * k2]);
    }
    std::vector<C> X(N);
    for (int k = 0; k < N; ++k) X[k] = y[k];
    auto yy = naive(X);
    for (int k2 = 0; k2 < 16; ++k2) {
        double2 v[N2];
        for (int n1 = 0; n1 < N2; ++n1) v[n1] = T2[n1][k2];
        dft<N2>(v);
        for (int k1 = 0; k1 < N2; ++k1) e = std::max(e, std::abs(cc(v[k1]) - yy[16 * k1 + k2]) / N);
    }
    return e;
}

int main() {
    double e[] = {test_block<2>(), test_block<3>(), test_block<4>(), test_block<8>(), test_block<12>(),
                  test_block<16>(), test_two_step<2>(), test_two_step<4>(), test_two_step<8>(),
                  test_two_step<12>(), test_two_step<16>()};
    const char* nm[] = {"dft2", "dft3", "dft4", "dft8", "dft12", "dft16", "N=32", "N=64", "N=128", "N=192", "N=256"};
    int bad = 0;
    for (int i = 0; i < 11; ++i) {
        printf("%-6s max err %.2e\n", nm[i], e[i]);
        bad += !(e[i] < 1e-12);
    }
    return bad;
}
