// Microbenchmark: tcgen05.mma kind::i8 issue rate from shared memory operands
// (SS mode), one CTA per SM, no TMA traffic.  Measures the per-SM ceiling the
// band GEMM can reach for M=128 and N in {128, 256}.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)(1024 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                 ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile("{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int N, int NACC>
__global__ void __launch_bounds__(128, 1) mma_kernel(int reps, int per_commit, long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, bar_end;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        mbar_init(&bar_end, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    if (warp == 0 && threadIdx.x == 0) {
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
        for (int r = 0; r < reps; r++) {
            for (int k = 0; k < 4; k++)
                mma_i8(tmem + (uint32_t)((r % NACC) * N), smem_desc(a0 + 32 * k), smem_desc(b0 + 32 * k), IDESC, (r > 0 || k > 0) ? 1u : 0u);
            if (per_commit && (r % per_commit) == per_commit - 1) {
                mma_commit(&bar);
            }
        }
        mma_commit(&bar_end);  // arrives when every MMA issued above has completed
    }
    __syncwarp();
    if (threadIdx.x == 0) mbar_wait(&bar_end, 0);
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}


// emulation of the band kernel's MMA-warp step: whole warp waits on two
// (already complete) mbarriers, fence, lane 0 issues PAIRS x 4 MMAs (N=256)
// and two commits, __syncwarp
template <int PAIRS, int ELECT_ALL>
__global__ void __launch_bounds__(128, 1) step_kernel(int steps, long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t done, c1, c2, bar_end;
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < (128 + 256) * 128 / 4; i += blockDim.x) ((uint32_t*)sm)[i] = i * 2654435761u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        mbar_init(&c1, 1);
        mbar_init(&c2, 1);
        mbar_init(&bar_end, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    if (warp == 0) {
        const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 128 * 128);
        for (int r = 0; r < steps; r++) {
            mbar_wait(&done, 0);
            mbar_wait(&done, 0);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            if (lane == 0) {
                for (int p = 0; p < PAIRS; p++)
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        mma_i8(tmem + (uint32_t)(p * 256), smem_desc(a0 + 32 * k), smem_desc(b0 + 32 * k), IDESC, 1u);
                mma_commit(&c1);
                mma_commit(&c2);
            }
            __syncwarp();
        }
        if (lane == 0) mma_commit(&bar_end);
        __syncwarp();
        mbar_wait(&bar_end, 0);
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int PAIRS>
void run_step(int steps) {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = (128 + 256) * 128 + 1024;
    cudaFuncSetAttribute(step_kernel<PAIRS, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    step_kernel<PAIRS, 0><<<148, 128, smem>>>(steps, d);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
    const double macs = 128.0 * 256 * 128.0 * PAIRS * steps;
    printf("step emulation PAIRS=%d steps=%d: %.0f cyc/step, %.0f MAC/clk/SM, err=%s\n", PAIRS, steps,
           (double)mx / steps, macs / mx, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

template <int N, int NACC>
void run(int reps, int per_commit) {
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    const int smem = (128 + N) * 128 + 1024;
    cudaFuncSetAttribute(mma_kernel<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    mma_kernel<N, NACC><<<148, 128, smem>>>(reps, per_commit, d);  // warm
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma_kernel<N, NACC><<<148, 128, smem>>>(reps, per_commit, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; i++) mx = h[i] > mx ? h[i] : mx;
    const double macs = 128.0 * N * 128.0 * reps;  // per CTA (4 MMAs of K=32 per rep)
    printf("N=%d nacc=%d reps=%d commit_every=%d: %.3f ms, %.0f MAC/clk/SM (clock64), %.2f POPS chip, err=%s\n", N, NACC,
           reps, per_commit, ms, macs / mx, 2 * macs * 148 / (ms * 1e-3) / 1e15, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<256, 2>(4096, 0);
    run<256, 2>(4096, 2);
    run<256, 1>(4096, 0);
    run<128, 4>(4096, 0);
    run<128, 4>(4096, 4);
    run_step<1>(2048);
    run_step<2>(2048);
    return 0;
}
