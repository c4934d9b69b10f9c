// fp64 throughput microbenchmark (dev tool): DMMA m8n8k4 and DFMA issue
// rates per SM at 1/2/4 warps per SM sub-partition, to pin the fp64
// roofline denominator the band solves are reported against.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(int iters, double* out) {
    double acc[CH][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c][0] = acc[c][1] = 0.0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) dmma(acc[c][0], acc[c][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) out[0] = s;
}

template <int CH>
__global__ void k_dfma(int iters, double* out) {
    double acc[CH];
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) acc[c] = fma(a, acc[c], b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += acc[c];
    if (s == 1.2345) out[0] = s;
}

// half the warps issue DMMA, half DFMA: do the two share one fp64 pipe?
__global__ void k_mixed(int iters, double* out) {
    const int warp = threadIdx.x >> 5;
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    double s = 0;
    if (warp & 1) {
        double acc[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = c;
        for (int i = 0; i < iters * 8; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = fma(a, acc[c], b);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) s += acc[c];
    } else {
        double acc[8][2];
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int c = 0; c < 8; ++c) dmma(acc[c][0], acc[c][1], a, b);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
    }
    if (s == 1.2345) out[0] = s;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    printf("{\"sms\": %d, \"runs\": [\n", nsm);
    bool first = true;
    for (int wps = 1; wps <= 8; wps *= 2) {
        const int threads = 128 * wps;
        for (int kind = 0; kind < 2; ++kind) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (kind == 0) k_dmma<8><<<nsm, threads>>>(iters, out);
                else k_dfma<8><<<nsm, threads>>>(iters, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
            }
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double warps = (double)nsm * threads / 32;
            const double flops = kind == 0 ? warps * iters * 8 * 512.0 : warps * iters * 8 * 64.0;
            printf("%s {\"kind\": \"%s\", \"warps_per_smsp\": %d, \"ms\": %.3f, \"tflops\": %.2f}",
                   first ? "" : ",\n", kind == 0 ? "dmma_m8n8k4" : "dfma", wps, ms,
                   flops / ms / 1e9);
            first = false;
        }
    }
    // dependent-chain latency: one warp per SM sub-partition, CH chains
    const int chs[] = {1, 2, 4, 8, 16};
    for (int ci = 0; ci < 5; ++ci) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            switch (chs[ci]) {
                case 1: k_dmma<1><<<nsm, 128>>>(iters, out); break;
                case 2: k_dmma<2><<<nsm, 128>>>(iters, out); break;
                case 4: k_dmma<4><<<nsm, 128>>>(iters, out); break;
                case 8: k_dmma<8><<<nsm, 128>>>(iters, out); break;
                default: k_dmma<16><<<nsm, 128>>>(iters, out); break;
            }
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        int clk = 0;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        const double per = ms * 1e-3 / ((double)iters * chs[ci]);
        printf(",\n {\"kind\": \"dmma_chains\", \"chains\": %d, \"ns_per_dmma_per_warp\": %.2f,"
               " \"latency_cycles_at_%d_mhz\": %.1f}", chs[ci], per * 1e9, clk / 1000,
               per * chs[ci] * clk * 1e3);
    }
    {
        // mixed: per SM 4 DMMA warps (iters x 8 DMMA) + 4 DFMA warps (8 iters x 8 DFMA)
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            k_mixed<<<nsm, 256>>>(iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl = (double)nsm * 4 * iters * 8 * 512.0 + (double)nsm * 4 * iters * 8 * 8 * 64.0;
        printf(",\n {\"kind\": \"mixed_dmma_dfma\", \"ms\": %.3f, \"tflops\": %.2f}", ms, fl / ms / 1e9);
    }
    printf("\n]}\n");
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(err)); return 1; }
    return 0;
}
