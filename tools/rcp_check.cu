// Accuracy of rcp.approx.ftz.f64 + k Newton steps vs IEEE 1/x (dev tool).
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = x[i], r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
    double ref = 1.0 / v;
    out[4 * i + 0] = fabs(r * v - 1.0);
    double e = fma(-v, r, 1.0); double r1 = fma(r, e, r);
    out[4 * i + 1] = fabs((r1 - ref) / ref);
    e = fma(-v, r1, 1.0); double r2 = fma(r1, e, r1);
    out[4 * i + 2] = fabs((r2 - ref) / ref);
    // cubic single step: r0 (1 + e + e^2), e = 1 - v r0
    double e0 = fma(-v, r, 1.0);
    double r3 = fma(r, fma(e0, e0, e0), r);
    out[4 * i + 3] = fabs((r3 - ref) / ref);
}
int main1() {
    const int n = 1 << 20;
    double *x, *o; cudaMallocManaged(&x, n * 8); cudaMallocManaged(&o, 4 * n * 8);
    unsigned long long s = 88172645463325252ull;
    for (int i = 0; i < n; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x[i] = 0.01 + 1000.0 * (double)(s >> 11) / 9007199254740992.0; }
    k<<<n / 256, 256>>>(x, o, n); cudaDeviceSynchronize();
    double m[4] = {0, 0, 0, 0};
    long nz2 = 0, nz3 = 0;
    for (int i = 0; i < n; i++) { for (int j = 0; j < 4; j++) m[j] = fmax(m[j], o[4 * i + j]); nz2 += o[4*i+2] != 0; nz3 += o[4*i+3] != 0; }
    printf("not correctly rounded: 2 NR %ld, cubic %ld of %d\n", nz2, nz3, n);
    printf("approx rel err %.3e, 1 NR %.3e, 2 NR %.3e, cubic %.3e (ulp=%.3e)\n", m[0], m[1], m[2], m[3], ldexp(1.0, -52));
    return 0;
}
// (appended) fsqrt accuracy check
__global__ void ks(const double* x, double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double v = x[i], y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    const double hx = 0.5 * v;
    const double y0 = y;
    y = y * fma(-hx * y, y, 1.5);
    const double s1 = v * y;                                   // one Newton step
    const double r1 = fma(fma(-s1, s1, v), 0.5 * y, s1);
    y = y * fma(-hx * y, y, 1.5);
    const double s = v * y;
    const double r = fma(fma(-s, s, v), 0.5 * y, s);
    const double ref = sqrt(v);
    out[3 * i + 0] = fabs(r - ref) / ref;
    out[3 * i + 1] = fabs(r1 - ref) / ref;
    out[3 * i + 2] = fabs(y0 * v - ref) / ref;                  // the hardware estimate
}
int main2() {
    const int n = 1 << 20;
    double *x, *o; cudaMallocManaged(&x, n * 8); cudaMallocManaged(&o, 3 * n * 8);
    unsigned long long s = 88172645463325252ull;
    for (int i = 0; i < n; i++) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        // log-uniform over 1e-8 .. 1e8 (g h + lam/3 sigma^2 of every config lies inside)
        x[i] = exp(log(1e-8) + (log(1e8) - log(1e-8)) * (double)(s >> 11) / 9007199254740992.0);
    }
    ks<<<n / 256, 256>>>(x, o, n); cudaDeviceSynchronize();
    double m[3] = {0, 0, 0}; long nz[2] = {0, 0};
    for (int i = 0; i < n; i++) for (int j = 0; j < 3; j++) m[j] = fmax(m[j], o[3 * i + j]);
    for (int i = 0; i < n; i++) { nz[0] += o[3 * i] != 0; nz[1] += o[3 * i + 1] != 0; }
    printf("fsqrt max rel err: 2 Newton %.3e (%ld not correctly rounded), 1 Newton %.3e (%ld), estimate %.3e (ulp %.3e)\n",
           m[0], nz[0], m[1], nz[1], m[2], ldexp(1.0, -52));
    return 0;
}
int main() { main1(); return main2(); }
