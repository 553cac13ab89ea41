// DFMA throughput microbenchmark (dev tool; SURVEY 8(d) asks for the measured
// fp64 peak, which MEASURED_PEAKS.json does not hold).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_peak tools/dfma_peak.cu && /tmp/dfma_peak
// Each thread runs 8 independent DFMA chains; grid = SMs x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double *out, int iters, double a, double b)
{
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = fma(x[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) s += x[k];
    if (s == 123.456) out[0] = s;   // keep the chains alive
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *out;
    cudaMalloc(&out, 8);
    const int threads = 256, blocks = sms * 8, iters = 1 << 16;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
    float best = 1e30f;
    for (int rep = 0; rep < 5; rep++) {
        cudaEventRecord(e0);
        dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double dfma = double(blocks) * threads * iters * 8;
    const double rate = dfma / (best * 1e-3);
    printf("{\"sms\": %d, \"max_clock_mhz\": %.0f, \"dfma_per_s\": %.4e, \"fp64_tflops\": %.2f, "
           "\"dfma_per_clk_per_sm_at_max_clock\": %.1f, \"ms\": %.3f}\n",
           sms, clk / 1e3, rate, 2.0 * rate / 1e12, rate / (sms * clk * 1e3), best);
    return 0;
}
