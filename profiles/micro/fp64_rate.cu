// fp64_rate.cu - B200 FP64 issue rate for the radius product's instruction mix:
// separate __dmul_rn / __dadd_rn (no contraction, as the reference's rounding
// sequence requires) vs fused __fma_rn, 16 independent chains per thread.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
    double s[16];
#pragma unroll
    for (int i = 0; i < 16; i++) s[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            // the product's operand comes from another chain (not loop-invariant)
            if (MODE == 0) s[i] = __dadd_rn(s[i], __dmul_rn(s[(i + 8) & 15], b));
            else s[i] = __fma_rn(s[(i + 8) & 15], b, s[i]);
        }
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) t += s[i];
    if (t == 12345.0) out[0] = t;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int threads = 256, iters = 4096;
    for (int occ : {1, 2, 4, 8}) {  // resident warps per SM = 8 * occ
    const int blocks = sms * occ;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters, 1.0000001, 0.5);
            else k<1><<<blocks, threads>>>(out, iters, 1.0000001, 0.5);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)blocks * threads * iters * 16 * (mode == 0 ? 2 : 1);  // instructions
            if (rep)
                printf("{\"mode\": \"%s\", \"warps_per_sm\": %d, \"ms\": %.3f, \"fp64_instr_per_s\": %.4g, \"per_sm_per_clk_at_1.965GHz\": %.2f}\n",
                       mode == 0 ? "dmul+dadd" : "fma", 8 * occ, ms, ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    }
    return 0;
}
