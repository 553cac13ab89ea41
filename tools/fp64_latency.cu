// fp64 latency / issue microbenchmark (dev tool): one CTA per SM, W warps per
// SM sub-partition, each thread running C independent dependent chains of one
// op; prints cycles per op per chain (C = 1, W = 1: the latency) and the SM's
// warp-instruction rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_lat tools/fp64_latency.cu && /tmp/fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP, int C>
__global__ void chain(double *out, long long *cyc, int iters, double a, double b)
{
    double x[C];
#pragma unroll
    for (int k = 0; k < C; k++) x[k] = threadIdx.x * 1e-3 + k + 1.0;
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < C; k++) {
            if (OP == 0) x[k] = fma(x[k], a, b);
            else if (OP == 1) x[k] = x[k] + b;
            else if (OP == 2) x[k] = x[k] * a;
            else {
                double r;
                asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[k]));
                x[k] = r;
            }
        }
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int k = 0; k < C; k++) s += x[k];
    if (s == 123.456) out[0] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP, int C>
void run(const char *name, int warps_per_sm, double *out, long long *cyc, int sms)
{
    const int iters = 4096;
    chain<OP, C><<<sms, 32 * warps_per_sm>>>(out, cyc, 64, 0.999999, 1e-7);
    chain<OP, C><<<sms, 32 * warps_per_sm>>>(out, cyc, iters, 0.999999, 1e-7);
    long long h = 0;
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per = double(h) / (double(iters) * C);
    printf("%-5s chains %d warps/SM %2d: %.2f cycles per op per chain, %.3f warp-instr/clk/SM\n", name, C,
           warps_per_sm, double(h) / iters, warps_per_sm / per);
}

int main()
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out;
    long long *cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * sms);
    for (int w : {4, 16, 32}) {
        run<0, 1>("DFMA", w, out, cyc, sms);
        run<0, 2>("DFMA", w, out, cyc, sms);
        run<0, 4>("DFMA", w, out, cyc, sms);
        run<1, 1>("DADD", w, out, cyc, sms);
        run<2, 1>("DMUL", w, out, cyc, sms);
        run<3, 1>("RCP64", w, out, cyc, sms);
        run<3, 4>("RCP64", w, out, cyc, sms);
    }
    return 0;
}
