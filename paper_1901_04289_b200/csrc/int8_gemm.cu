// int8_gemm.cu - K5: exact scaled-integer block product on the 5th-gen tensor
// cores (tcgen05 kind::i8, TMA-fed, int32 accumulators in TMEM).
//
// Replaces int_matmul_multimodular (src/matmul.cpp:280-350, paths relative to
// /root/reference/proj): instead of residues mod 61-bit primes and a CRT, the
// scaled integers a_ik (height <= H_A bits) and b_kj are cut into balanced
// signed 8-bit digits, a = sum_s A_s 256^s, b = sum_t B_t 256^t (scale_pack in
// matmul.cu), and
//     T_ij = sum_d 256^d D_d,   D_d = sum_{s+t=d} (A_s B_t)_ij .
// Each diagonal D_d (or a chunk of its slice pairs, bounded so |D| < 2^30)
// is accumulated exactly in an int32 TMEM tile by tcgen05.mma over K; the
// epilogue warps stream the diagonals in increasing d with a per-entry carry:
//     v = carry + D_d ;  byte_d = v mod 256 ;  carry = v >> 8
// so each byte is final when emitted.  Bytes are packed 4 per uint32 word
// (Tw[word][row][col]); each CTA covers one 128x128 output tile and one group
// of consecutive diagonals (group boundaries are multiples of 4), and leaves
// its final carry in Tc[group][row][col].  The recombine kernel forms
// T = (bytes as an unsigned number) + sum_g Tc[g] 256^(d1_g).
//
// Roles (320 threads): warp 0 TMA producer, warp 1 MMA issuer (one lane),
// warps 2..9 epilogue (two warps per TMEM lane quarter, 64 columns each).
// Shapes: UMMA M=128, N=128, K=32 (int8); smem tiles 128x128 B with the
// 128-byte swizzle; 4-stage smem ring; 2 TMEM accumulator buffers.

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "apb.h"
#include "apb_internal.h"
#include "int8_gemm.h"

namespace apb {

namespace {

constexpr int BM = 128, BN = 128, BK = 128;  // BK in bytes (= int8 elements)
constexpr int STAGES = 4;
constexpr int STAGE_A = BM * BK, STAGE_B = BN * BK;
constexpr int STAGE_BYTES = STAGE_A + STAGE_B;
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 32 * (2 + EPI_WARPS);
constexpr int TMEM_COLS = 256;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// K-major, 128-byte swizzle smem matrix descriptor (8-row atoms of 1024 B)
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)(1024 >> 4) << 32;  // stride byte offset between 8-row groups
    d |= (uint64_t)1 << 46;            // sm100 descriptor version
    d |= (uint64_t)2 << 61;            // SWIZZLE_128B
    return d;
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}

#define TMEM_LD32(taddr, v)                                                                      \
    asm volatile(                                                                                \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"       \
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),             \
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),          \
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),          \
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),          \
          "=r"(v[31])                                                                            \
        : "r"(taddr))

#define TMEM_ST32(taddr, v)                                                                      \
    asm volatile(                                                                                \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"          \
        ::"r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), \
          "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]),        \
          "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]),      \
          "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),      \
          "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])                                           \
        : "memory")

// instruction descriptor: s32 accumulate, s8 x s8, K-major both, M=128, N=128
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                            ((uint32_t)(BM >> 4) << 24);

__global__ void __launch_bounds__(THREADS, 1)
    slice_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      SliceGemmParams P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t* bars = (uint64_t*)(smem + STAGES * STAGE_BYTES);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* tfull = bars + 2 * STAGES;
    uint64_t* tempty = bars + 2 * STAGES + 2;
    uint32_t* tmem_slot = (uint32_t*)(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = blockIdx.x;   // diagonal group
    const int mt = blockIdx.y;  // row tile
    const int nt = blockIdx.z;  // col tile
    const int m0 = mt * BM, n0 = nt * BN;
    const int u_begin = P.group_unit_begin[g], u_end = P.group_unit_begin[g + 1];

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], EPI_WARPS * 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            int stage = 0;
            uint32_t phase = 0;
            for (int u = u_begin; u < u_end; u++) {
                const int4 U = P.units[u];  // (d, s_lo, s_hi, flags)
                for (int s = U.y; s < U.z; s++) {
                    const int t = U.x - s;
                    for (int kb = 0; kb < P.n_kb; kb++) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * STAGE_BYTES;
                        mbar_expect_tx(&full[stage], STAGE_BYTES);
                        tma_load_2d(sa, &tmA, kb * BK, s * P.Mp + m0, &full[stage]);
                        tma_load_2d(sa + STAGE_A, &tmB, kb * BK, t * P.Np + n0, &full[stage]);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        int stage = 0;
        uint32_t phase = 0;
        for (int u = u_begin; u < u_end; u++) {
            const int ui = u - u_begin;
            const int buf = ui & 1;
            const uint32_t tph = (ui >> 1) & 1;
            const int4 U = P.units[u];
            mbar_wait(&tempty[buf], tph ^ 1);
            fence_after();
            const uint32_t tmem_d = tmem_base + (uint32_t)(buf * BN);
            uint32_t acc = 0;
            for (int s = U.y; s < U.z; s++) {
                for (int kb = 0; kb < P.n_kb; kb++) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(smem + stage * STAGE_BYTES);
                        const uint32_t b0 = a0 + STAGE_A;
#pragma unroll
                        for (int k = 0; k < BK / 32; k++) {
                            mma_i8(tmem_d, smem_desc(a0 + 32 * k), smem_desc(b0 + 32 * k), kIdesc, acc);
                            acc = 1;
                        }
                        mma_commit(&empty[stage]);
                    }
                    __syncwarp();
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
            if (lane == 0) mma_commit(&tfull[buf]);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------ epilogue
        const int e = warp - 2;
        const int q = warp & 3;          // TMEM lane quarter this warp may access
        const int col0 = (e >> 2) * 64;  // column half
        const int row = m0 + 32 * q + lane;
        int32_t carry[64];
        uint32_t word[64];
#pragma unroll
        for (int c = 0; c < 64; c++) {
            carry[c] = 0;
            word[c] = 0;
        }
        for (int u = u_begin; u < u_end; u++) {
            const int ui = u - u_begin;
            const int buf = ui & 1;
            const uint32_t tph = (ui >> 1) & 1;
            const int4 U = P.units[u];
            const int d = U.x;
            const bool first = (U.w & 1) != 0, last = (U.w & 2) != 0;
            mbar_wait(&tfull[buf], tph);
            fence_after();
            uint32_t v[64];
            const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(buf * BN + col0);
            TMEM_LD32(taddr, v);
            TMEM_LD32(taddr + 32, (v + 32));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            fence_before();
            mbar_arrive(&tempty[buf]);
            const int sh = 8 * (d & 3);
#pragma unroll
            for (int c = 0; c < 64; c++) {
                const int32_t D = (int32_t)v[c];
                const int32_t b = (int32_t)((word[c] >> sh) & 255u);
                const int32_t val = b + D + (first ? carry[c] : 0);
                word[c] = (word[c] & ~(255u << sh)) | ((uint32_t)(val & 255) << sh);
                carry[c] = (first ? 0 : carry[c]) + (val >> 8);
            }
            if (last && ((d & 3) == 3 || d == P.group_d1[g] - 1)) {
                uint32_t* dst = P.Tw + ((size_t)(d >> 2) * P.Mp + row) * P.Np + n0 + col0;
#pragma unroll
                for (int c = 0; c < 64; c += 4) {
                    *(uint4*)(dst + c) = make_uint4(word[c], word[c + 1], word[c + 2], word[c + 3]);
                    word[c] = word[c + 1] = word[c + 2] = word[c + 3] = 0;
                }
            }
        }
        int32_t* cdst = P.Tc + ((size_t)g * P.Mp + row) * P.Np + n0 + col0;
#pragma unroll
        for (int c = 0; c < 64; c += 4)
            *(int4*)(cdst + c) = make_int4(carry[c], carry[c + 1], carry[c + 2], carry[c + 3]);
    }

    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
    }
}


// ====================================================================
// Band kernel: 4 consecutive diagonals per pass.  For one output tile and a
// band d0..d0+3, every A slice s and every B slice t of the band is loaded
// ONCE per K block and feeds up to 4 MMAs (one per diagonal accumulator),
// which cuts the L2->SMEM operand traffic ~4x against one diagonal at a time.
// Sweep per K block: s descending from s_hi to s_lo; the live B slices form a
// sliding window t in [max(0,d0-s), min(S_B-1,d0+3-s)] that advances by one
// slice per step (FIFO ring).  Accumulators: 4 x 128 TMEM columns (512).
// Each (tile, band) work item is independent (carry-in 0, carry-out to
// Tc[band]); items are LPT-assigned to persistent CTAs on the host.
// Requires |D_d| < 2^31: pairs(d) * K * 2^14 < 2^31 (checked by the driver).
// variants: <BNT=128, W=4> (4 diagonals, N=128 MMAs) and <BNT=256, W=2>
// (2 diagonals, N=256 MMAs: half the MMA issues per unit of work)
template <int BNT, int W>
struct BandCfg {
    static constexpr int A_STAGES = 4;
    static constexpr int TILE_A = 128 * BK;
    static constexpr int TILE_B = BNT * BK;
#ifndef APB_BAND_BSTAGES
#define APB_BAND_BSTAGES 4
#endif
    // 4 B stages at BNT=256 leave ~34 KB of shared memory for a co-resident radius block
    static constexpr int B_STAGES = BNT == 128 ? 8 : APB_BAND_BSTAGES;
    static constexpr int SMEM = A_STAGES * TILE_A + B_STAGES * TILE_B + 1024 + 512;
    static constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BNT >> 3) << 17) |
                                      ((uint32_t)(BM >> 4) << 24);
};

template <int BNT, int BAND_W>
__global__ void __launch_bounds__(THREADS, 1)
    band_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     BandGemmParams P) {
    using Cfg = BandCfg<BNT, BAND_W>;
    constexpr int A_STAGES = Cfg::A_STAGES, B_STAGES = Cfg::B_STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* smA = smem;
    uint8_t* smB = smem + A_STAGES * Cfg::TILE_A;
    uint64_t* bars = (uint64_t*)(smem + A_STAGES * Cfg::TILE_A + B_STAGES * Cfg::TILE_B);
    uint64_t* fullA = bars;
    uint64_t* emptyA = fullA + A_STAGES;
    uint64_t* fullB = emptyA + A_STAGES;
    uint64_t* emptyB = fullB + B_STAGES;
    uint64_t* tfull = emptyB + B_STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it_begin = P.cta_begin[blockIdx.x], it_end = P.cta_begin[blockIdx.x + 1];
    if (P.dbg_ts && threadIdx.x == 0) P.dbg_ts[blockIdx.x * 32 + 31] = clock64();

    if (threadIdx.x == 0) {
        for (int i = 0; i < A_STAGES; i++) {
            mbar_init(&fullA[i], 1);
            mbar_init(&emptyA[i], 1);
        }
        for (int i = 0; i < B_STAGES; i++) {
            mbar_init(&fullB[i], 1);
            mbar_init(&emptyB[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, EPI_WARPS * 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            uint32_t ai = 0, bi = 0;  // sequential ring indices
            for (int it = it_begin; it < it_end; it++) {
                const int2 W = P.items[it];
                const int m0 = (W.x / P.n_tiles_n) * 128, n0 = (W.x % P.n_tiles_n) * BNT;
                const int d0 = BAND_W * W.y;
                const int s_hi = min(P.S_A - 1, d0 + BAND_W - 1), s_lo = max(0, d0 - (P.S_B - 1));
                for (int kb = 0; kb < P.n_kb; kb++) {
                    int tmax_prev = -1;
                    for (int s = s_hi; s >= s_lo; s--) {
                        const int tmin = max(0, d0 - s), tmax = min(P.S_B - 1, d0 + BAND_W - 1 - s);
                        {
                            const uint32_t st = ai % A_STAGES, ph = (ai / A_STAGES) & 1;
                            mbar_wait(&emptyA[st], ph ^ 1);
                            if ((P.debug & 1) && ai >= (uint32_t)A_STAGES) {
                                mbar_arrive(&fullA[st]);
                            } else {
                                mbar_expect_tx(&fullA[st], Cfg::TILE_A);
                                tma_load_2d(smA + st * Cfg::TILE_A, &tmA, kb * BK, s * P.Mp + m0, &fullA[st]);
                            }
                            ai++;
                        }
                        for (int t = max(tmin, tmax_prev + 1); t <= tmax; t++) {
                            const uint32_t st = bi % B_STAGES, ph = (bi / B_STAGES) & 1;
                            mbar_wait(&emptyB[st], ph ^ 1);
                            if ((P.debug & 1) && bi >= (uint32_t)B_STAGES) {
                                mbar_arrive(&fullB[st]);
                            } else {
                                mbar_expect_tx(&fullB[st], Cfg::TILE_B);
                                tma_load_2d(smB + st * Cfg::TILE_B, &tmB, kb * BK, t * P.Np + n0, &fullB[st]);
                            }
                            bi++;
                        }
                        tmax_prev = tmax;
                    }
                }
            }
        }
    } else if (warp == 1) {
        uint32_t ai = 0, bi = 0;
        uint32_t tph = 0;
        for (int it = it_begin; it < it_end; it++) {
            const int2 W = P.items[it];
            const int d0 = BAND_W * W.y;
            const int s_hi = min(P.S_A - 1, d0 + BAND_W - 1), s_lo = max(0, d0 - (P.S_B - 1));
            if (P.dbg_ts && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 0] = clock64();
            mbar_wait(tempty, tph ^ 1);
            fence_after();
            if (P.dbg_ts && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 1] = clock64();
            uint32_t init_mask = 0;
            for (int kb = 0; kb < P.n_kb; kb++) {
                const int t_first = max(0, d0 - s_hi);
                const uint32_t b_first = bi;  // ring index of B slice t_first in this sweep
                int tmax_prev = -1;
                for (int s = s_hi; s >= s_lo; s--) {
                    const int tmin = max(0, d0 - s), tmax = min(P.S_B - 1, d0 + BAND_W - 1 - s);
                    const uint32_t ast = ai % A_STAGES, aph = (ai / A_STAGES) & 1;
                    mbar_wait(&fullA[ast], aph);
                    for (int t = max(tmin, tmax_prev + 1); t <= tmax; t++) {
                        const uint32_t bidx = b_first + (uint32_t)(t - t_first);
                        mbar_wait(&fullB[bidx % B_STAGES], (bidx / B_STAGES) & 1);
                    }
                    fence_after();
                    if (lane == 0) {
                        const uint32_t a0 = smem_u32(smA + ast * Cfg::TILE_A);
                        for (int t = tmin; t <= tmax; t++) {
                            const int w = s + t - d0;
                            const uint32_t bidx = b_first + (uint32_t)(t - t_first);
                            const uint32_t b0 = smem_u32(smB + (bidx % B_STAGES) * Cfg::TILE_B);
                            const uint32_t tmem_d = tmem_base + (uint32_t)(w * BNT);
#pragma unroll
                            for (int k = 0; k < BK / 32; k++) {
                                const uint32_t acc = ((init_mask >> w) & 1u) | (k > 0 ? 1u : 0u);
                                mma_i8(tmem_d, smem_desc(a0 + 32 * k), smem_desc(b0 + 32 * k), Cfg::IDESC, acc);
                            }
                            init_mask |= 1u << w;
                        }
                        mma_commit(&emptyA[ast]);
                        if (s > s_lo) {
                            const int tr = d0 - s;  // last use of slice tr is at this s
                            if (tr >= 0) {
                                const uint32_t bidx = b_first + (uint32_t)(tr - t_first);
                                mma_commit(&emptyB[bidx % B_STAGES]);
                            }
                        } else {
                            for (int t = tmin; t <= tmax; t++) {
                                const uint32_t bidx = b_first + (uint32_t)(t - t_first);
                                mma_commit(&emptyB[bidx % B_STAGES]);
                            }
                        }
                    }
                    __syncwarp();
                    ai++;
                    tmax_prev = tmax;
                }
                bi = b_first + (uint32_t)(min(P.S_B - 1, d0 + BAND_W - 1 - s_lo) - t_first + 1);
            }
            if (lane == 0) mma_commit(tfull);
            if (P.dbg_ts && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 2] = clock64();
            __syncwarp();
            tph ^= 1;
        }
    } else {
        const int e = warp - 2;
        const int q = warp & 3;
        const int col0 = (e >> 2) * (BNT / 2);
        uint32_t tph = 0;
        for (int it = it_begin; it < it_end; it++) {
            const int2 W = P.items[it];
            const int m0 = (W.x / P.n_tiles_n) * 128, n0 = (W.x % P.n_tiles_n) * BNT;
            const int d0 = BAND_W * W.y;
            const int row = m0 + 32 * q + lane;
            mbar_wait(tfull, tph);
            fence_after();
            if (P.dbg_ts && warp == 2 && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 3] = clock64();
#pragma unroll 1
            for (int h = 0; h < BNT / 64; h++) {
                int32_t carry[32];
                uint32_t word[32];
#pragma unroll
                for (int c = 0; c < 32; c++) {
                    carry[c] = 0;
                    word[c] = 0;
                }
#pragma unroll 1
                for (int w = 0; w < BAND_W; w++) {
                    // diagonals past the last one contribute D = 0, so every band's
                    // carry leaves at bit 32 (b + 1) (word aligned for the recombine)
                    uint32_t v[32];
                    if (d0 + w < P.ND) {
                        const uint32_t taddr = tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(w * BNT + col0 + 32 * h);
                        TMEM_LD32(taddr, v);
                        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; c++) v[c] = 0;
                    }
#pragma unroll
                    for (int c = 0; c < 32; c++) {
                        const int64_t val = (int64_t)(int32_t)v[c] + carry[c];
                        word[c] |= (uint32_t)(val & 255) << (8 * w);
                        carry[c] = (int32_t)(val >> 8);
                    }
                }
                // quad layout plane[band][col/4][row][col%4]: the 32 lanes (rows) of a
                // warp store 512 contiguous bytes per instruction
                const size_t q0 = (size_t)W.y * (P.Np >> 2) + ((size_t)(n0 + col0 + 32 * h) >> 2);
                if (!(P.debug & 2)) {
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const size_t off = (((q0 + (c >> 2)) * P.Mp + row) << 2);
                        *(uint4*)(P.Tw + off) = make_uint4(word[c], word[c + 1], word[c + 2], word[c + 3]);
                        *(int4*)(P.Tc + off) = make_int4(carry[c], carry[c + 1], carry[c + 2], carry[c + 3]);
                    }
                }
            }
            fence_before();
            if (P.dbg_ts && warp == 2 && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 4] = clock64();
            mbar_arrive(tempty);
            tph ^= 1;
        }
    }

    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                     : "memory");
    }
}

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// span timer: every CTA folds its entry time into a min and its exit time into
// a max; the last CTA to leave adds the span to the running sum and resets
__device__ __forceinline__ void span_timer_enter(unsigned long long* T) {
    if (T && threadIdx.x == 0) atomicMin(&T[2], globaltimer());
}
__device__ __forceinline__ void span_timer_exit(unsigned long long* T) {
    if (T && threadIdx.x == 0) {
        atomicMax(&T[4], globaltimer());
        __threadfence();
        if (atomicAdd(&T[3], 1ull) == gridDim.x - 1) {
            __threadfence();
            const unsigned long long t0 = atomicAdd(&T[2], 0ull), t1 = atomicAdd(&T[4], 0ull);
            T[0] += t1 - t0;
            T[1] += 1;
            T[2] = ~0ull;
            T[3] = 0;
            T[4] = 0;
            __threadfence();
        }
    }
}

// ====================================================================
// Band kernel v3: same work decomposition and output as band_gemm_kernel, with
// a leaner MMA issue path (the v2 profile showed the single MMA thread, not the
// tensor pipe, setting the pace: ~270 warp instructions and 3-4 mbarrier waits
// per sweep step).
//  * one "step" barrier pair per A-ring slot: the producer posts the A tile
//    and every new B tile of step j on full[j % RA] (one expect_tx), the MMA
//    thread commits step j to empty[j % RA]; a B slot is recycled once the
//    last step that read its previous tile has completed (tracked by the
//    producer, which waits on that step's empty barrier);
//  * the MMA loop runs on one thread with smem descriptors advanced by adds;
//  * the epilogue issues all of a column chunk's TMEM loads before one wait.
// K blocks between normalisations for an item whose sweep has `pairs` A slices:
// each diagonal gains at most pairs * 128 * 2^14 per K block (0 = never needed)
__device__ __forceinline__ int item_kb_norm(const BandGemmParams& P, int pairs) {
    if (!P.kb_norm) return 0;
    const int lim = (int)((((int64_t)1 << 17) - 1) / ((int64_t)pairs * BK));
    const int k = min(P.kb_norm, lim);
    return k >= P.n_kb ? 0 : max(k, 1);
}

#ifndef APB_BAND_MAXNREG
#define APB_BAND_MAXNREG 168
#endif
// register cap (168 = the most 10 warps fit: 3 warps per SM sub-partition); 144 leaves room on every SM sub-partition for a co-resident 4-warp
// radius block (APB_RAD_BESIDE schedule), at the price of epilogue spills
// RAW: raw-accumulator epilogue (P.raw), a pure TMEM -> global copy: 128 registers, which
// leaves every SM sub-partition (3 of these warps each) room for one 128-register warp of the
// radius kernel launched beside it
template <int BNT, int BAND_W, bool RAW, bool SPLIT = false>
__global__ void __maxnreg__(BNT == 256 ? (RAW ? 128 : APB_BAND_MAXNREG) : 168)
    band3_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                      BandGemmParams P) {
    using Cfg = BandCfg<BNT, BAND_W>;
    constexpr int RA = Cfg::A_STAGES, RB = Cfg::B_STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* smA = smem;
    uint8_t* smB = smem + RA * Cfg::TILE_A;
    uint64_t* bars = (uint64_t*)(smem + RA * Cfg::TILE_A + RB * Cfg::TILE_B);
    uint64_t* full = bars;
    uint64_t* empty = full + RA;
    uint64_t* tfull = empty + RA;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 1);

    if (P.spec_maxw && ((int)((P.spec_maxw[0] + 9) / 8) != P.S_A || (int)((P.spec_maxw[1] + 9) / 8) != P.S_B))
        return;  // speculation void: the host redoes the product
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int it_begin = P.cta_begin[blockIdx.x], it_end = P.cta_begin[blockIdx.x + 1];
    if (P.dbg_ts && threadIdx.x == 0) P.dbg_ts[blockIdx.x * 32 + 31] = clock64();
    span_timer_enter(P.timer);
    // a programmatic dependent (the sparse radius products, which do not read this grid's
    // output) may be scheduled beside these CTAs once every one of them is resident
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (threadIdx.x == 0) {
        for (int i = 0; i < RA; i++) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, EPI_WARPS * 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
            int lastuse[RB];
#pragma unroll
            for (int q = 0; q < RB; q++) lastuse[q] = -1;
            int j = 0;        // step counter
            uint32_t bi = 0;  // B ring sequence index
            for (int it = it_begin; it < it_end; it++) {
                const int2 W = P.items[it];
                const int m0 = (W.x / P.n_tiles_n) * 128, n0 = (W.x % P.n_tiles_n) * BNT;
                const int d0 = BAND_W * (SPLIT ? (W.y & 0xFFFF) : W.y);
                const int kb0 = SPLIT ? (W.y >> 16) * P.kb_per : 0;
                const int kb1 = SPLIT ? min(P.n_kb, kb0 + P.kb_per) : P.n_kb;
                const int s_hi = min(P.S_A - 1, d0 + BAND_W - 1), s_lo = max(0, d0 - (P.S_B - 1));
                for (int kb = SPLIT ? kb0 : 0; kb < (SPLIT ? kb1 : P.n_kb); kb++) {
                    const int t_first = max(0, d0 - s_hi);
                    const uint32_t b_first = bi;
                    int tmax_prev = -1;
                    for (int s = s_hi; s >= s_lo; s--, j++) {
                        const int tmin = max(0, d0 - s), tmax = min(P.S_B - 1, d0 + BAND_W - 1 - s);
                        const int slot = j % RA;
                        if (j >= RA) mbar_wait(&empty[slot], ((j / RA) & 1) ^ 1);  // step j - RA done
                        const int tnew = max(tmin, tmax_prev + 1);
                        // recycled B slots: the step that last read the old tile must be done
                        for (int t = tnew; t <= tmax; t++) {
                            const int bs = (int)((b_first + (uint32_t)(t - t_first)) % RB);
                            int L = -1;
#pragma unroll
                            for (int q = 0; q < RB; q++)
                                if (q == bs) L = lastuse[q];
                            if (L >= 0 && L > j - RA) mbar_wait(&empty[L % RA], (L / RA) & 1);
                        }
                        mbar_expect_tx(&full[slot], Cfg::TILE_A + (uint32_t)(tmax - tnew + 1) * Cfg::TILE_B);
                        tma_load_2d(smA + slot * Cfg::TILE_A, &tmA, kb * BK, s * P.Mp + m0, &full[slot]);
                        for (int t = tnew; t <= tmax; t++) {
                            const int bs = (int)((b_first + (uint32_t)(t - t_first)) % RB);
                            tma_load_2d(smB + bs * Cfg::TILE_B, &tmB, kb * BK, t * P.Np + n0, &full[slot]);
                        }
                        for (int t = tmin; t <= tmax; t++) {
                            const int bs = (int)((b_first + (uint32_t)(t - t_first)) % RB);
#pragma unroll
                            for (int q = 0; q < RB; q++)
                                if (q == bs) lastuse[q] = j;
                        }
                        tmax_prev = tmax;
                    }
                    bi = b_first + (uint32_t)(min(P.S_B - 1, d0 + BAND_W - 1 - s_lo) - t_first + 1);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint64_t a_desc0 = smem_desc(smem_u32(smA)), b_desc0 = smem_desc(smem_u32(smB));
            int j = 0;
            uint32_t bi = 0, tph = 0;
            for (int it = it_begin; it < it_end; it++) {
                const int2 W = P.items[it];
                const int d0 = BAND_W * (SPLIT ? (W.y & 0xFFFF) : W.y);
                const int kb0 = SPLIT ? (W.y >> 16) * P.kb_per : 0;
                const int kb1 = SPLIT ? min(P.n_kb, kb0 + P.kb_per) : P.n_kb;
                const int s_hi = min(P.S_A - 1, d0 + BAND_W - 1), s_lo = max(0, d0 - (P.S_B - 1));
                if (P.dbg_ts && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 0] = clock64();
                mbar_wait(tempty, tph ^ 1);
                fence_after();
                if (P.dbg_ts && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 1] = clock64();
                uint32_t init_mask = 0;
                const int kbn = RAW ? 0 : item_kb_norm(P, s_hi - s_lo + 1);
                for (int kb = SPLIT ? kb0 : 0; kb < (SPLIT ? kb1 : P.n_kb); kb++) {
                    const int t_first = max(0, d0 - s_hi);
                    const uint32_t b_first = bi;
                    for (int s = s_hi; s >= s_lo; s--, j++) {
                        const int tmin = max(0, d0 - s), tmax = min(P.S_B - 1, d0 + BAND_W - 1 - s);
                        const int slot = j % RA;
                        mbar_wait(&full[slot], (j / RA) & 1);
                        fence_after();
                        const uint64_t ad = a_desc0 + (uint64_t)((slot * Cfg::TILE_A) >> 4);
                        for (int t = tmin; t <= tmax; t++) {
                            const int w = s + t - d0;
                            const int bs = (int)((b_first + (uint32_t)(t - t_first)) % RB);
                            const uint64_t bd = b_desc0 + (uint64_t)((bs * Cfg::TILE_B) >> 4);
                            const uint32_t td = tmem_base + (uint32_t)(w * BNT);
                            const uint32_t acc0 = (init_mask >> w) & 1u;
                            mma_i8(td, ad, bd, Cfg::IDESC, acc0);
#pragma unroll
                            for (int k = 1; k < BK / 32; k++) mma_i8(td, ad + 2 * k, bd + 2 * k, Cfg::IDESC, 1u);
                            init_mask |= 1u << w;
                        }
                        mma_commit(&empty[slot]);
                    }
                    bi = b_first + (uint32_t)(min(P.S_B - 1, d0 + BAND_W - 1 - s_lo) - t_first + 1);
                    if (kbn && (kb + 1) % kbn == 0 && kb + 1 < P.n_kb) {
                        // the epilogue folds the accumulators back to [0, 256) before more K
                        mma_commit(tfull);
                        tph ^= 1;
                        mbar_wait(tempty, tph ^ 1);
                        fence_after();
                    }
                }
                mma_commit(tfull);
                if (P.dbg_ts && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 2] = clock64();
                tph ^= 1;
            }
        }
    } else {
        const int e = warp - 2;
        const int q = warp & 3;
        const int col0 = (e >> 2) * (BNT / 2);
        uint32_t tph = 0;
        for (int it = it_begin; it < it_end; it++) {
            const int2 W = P.items[it];
            const int m0 = (W.x / P.n_tiles_n) * 128, n0 = (W.x % P.n_tiles_n) * BNT;
            const int d0 = BAND_W * (SPLIT ? (W.y & 0xFFFF) : W.y);
            const int row = m0 + 32 * q + lane;
            const int kbn = RAW ? 0 : item_kb_norm(P, min(P.S_A - 1, d0 + BAND_W - 1) - max(0, d0 - (P.S_B - 1)) + 1);
            const int n_norm = kbn ? (P.n_kb - 1) / kbn : 0;
            for (int ev = 0; ev < n_norm; ev++) {
                // in-place normalisation: D_w = r_w + 256 q_w, r_w in [0, 256); q_w moves to
                // D_{w+1} (weight 256), the top q to the band's carry (Tc, accumulated here)
                mbar_wait(tfull, tph);
                fence_after();
#pragma unroll 1
                for (int h = 0; h < BNT / 64; h++) {
                    int32_t cq[32];
#pragma unroll
                    for (int c = 0; c < 32; c++) cq[c] = 0;
#pragma unroll
                    for (int w0 = 0; w0 < BAND_W; w0++) {
                        // a diagonal past the last one is never accumulated by the MMAs: its
                        // region starts at 0 here and keeps the residue passed through it
                        uint32_t v[32];
                        const uint32_t taddr =
                            tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(w0 * BNT + col0 + 32 * h);
                        if (d0 + w0 < P.ND || ev) {
                            TMEM_LD32(taddr, v);
                            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                        } else {
#pragma unroll
                            for (int c = 0; c < 32; c++) v[c] = 0;
                        }
#pragma unroll
                        for (int c = 0; c < 32; c++) {
                            const int32_t val = (int32_t)v[c] + cq[c];
                            v[c] = (uint32_t)(val & 255);
                            cq[c] = val >> 8;
                        }
                        TMEM_ST32(taddr, v);
                    }
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    const size_t q0 = (size_t)W.y * (P.Np >> 2) + ((size_t)(n0 + col0 + 32 * h) >> 2);
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const size_t off = (((q0 + (c >> 2)) * P.Mp + row) << 2);
                        int4 t = ev ? *(int4*)(P.Tc + off) : make_int4(0, 0, 0, 0);
                        t.x += cq[c];
                        t.y += cq[c + 1];
                        t.z += cq[c + 2];
                        t.w += cq[c + 3];
                        *(int4*)(P.Tc + off) = t;
                    }
                }
                fence_before();
                mbar_arrive(tempty);
                tph ^= 1;
            }
            mbar_wait(tfull, tph);
            fence_after();
            if (P.dbg_ts && warp == 2 && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 3] = clock64();
            if (RAW) {
                // raw epilogue: the int32 accumulators go out as they are (plane Tw = the band's
                // first diagonal, Tc = its second); the accumulators are free once the last
                // chunk is in registers, so the next item's MMAs start under the final stores
#pragma unroll 1
                for (int h = 0; h < BNT / 64; h++) {
                    uint32_t v[2][32];
#pragma unroll
                    for (int u = 0; u < 2; u++) {
                        if (d0 + u < P.ND) {
                            const uint32_t taddr =
                                tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)(u * BNT + col0 + 32 * h);
                            TMEM_LD32(taddr, v[u]);
                        } else {
#pragma unroll
                            for (int c = 0; c < 32; c++) v[u][c] = 0;
                        }
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    if (h == BNT / 64 - 1) {
                        fence_before();
                        mbar_arrive(tempty);
                    }
                    const size_t q0 = (size_t)(SPLIT ? (W.y & 0xFFFF) + (W.y >> 16) * P.n_bands : W.y) * (P.Np >> 2) +
                                      ((size_t)(n0 + col0 + 32 * h) >> 2);
                    if (P.raw == 2) {
                        // 40-bit band values V = D0 + 256 D1 (|V| < 2^39 on this path): low words in Tw,
                        // the four high bytes of a column quad in one word of the byte plane Tc
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            uint32_t lo[4], hi = 0;
#pragma unroll
                            for (int e = 0; e < 4; e++) {
                                const int64_t V = (int64_t)(int32_t)v[1][c + e] * 256 + (int64_t)(int32_t)v[0][c + e];
                                lo[e] = (uint32_t)V;
                                hi |= ((uint32_t)(V >> 32) & 0xFFu) << (8 * e);
                            }
                            const size_t qe = (q0 + (c >> 2)) * P.Mp + row;
                            *(uint4*)(P.Tw + (qe << 2)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                            ((uint32_t*)P.Tc)[qe] = hi;
                        }
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; c += 4) {
                            const size_t off = (((q0 + (c >> 2)) * P.Mp + row) << 2);
                            *(uint4*)(P.Tw + off) = make_uint4(v[0][c], v[0][c + 1], v[0][c + 2], v[0][c + 3]);
                            *(uint4*)(P.Tc + off) = make_uint4(v[1][c], v[1][c + 1], v[1][c + 2], v[1][c + 3]);
                        }
                    }
                }
                if (P.dbg_ts && warp == 2 && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 4] = clock64();
                tph ^= 1;
                continue;
            }
            constexpr int WB = BAND_W == 2 ? 2 : 1;  // TMEM loads in flight per wait
#pragma unroll 1
            for (int h = 0; h < BNT / 64; h++) {
                int32_t carry[32];
                uint32_t word[32];
#pragma unroll
                for (int c = 0; c < 32; c++) {
                    carry[c] = 0;
                    word[c] = 0;
                }
#pragma unroll
                for (int w0 = 0; w0 < BAND_W; w0 += WB) {
                    uint32_t v[WB][32];
#pragma unroll
                    for (int u = 0; u < WB; u++) {
                        // diagonals past the last one contribute D = 0, so every band's
                        // carry leaves at the band boundary (word aligned for the recombine)
                        if (d0 + w0 + u < P.ND || n_norm) {
                            const uint32_t taddr =
                                tmem_base + ((uint32_t)(32 * q) << 16) + (uint32_t)((w0 + u) * BNT + col0 + 32 * h);
                            TMEM_LD32(taddr, v[u]);
                        } else {
#pragma unroll
                            for (int c = 0; c < 32; c++) v[u][c] = 0;
                        }
                    }
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                    for (int u = 0; u < WB; u++)
#pragma unroll
                        for (int c = 0; c < 32; c++) {
                            const int64_t val = (int64_t)(int32_t)v[u][c] + carry[c];
                            word[c] |= (uint32_t)(val & 255) << (8 * (w0 + u));
                            carry[c] = (int32_t)(val >> 8);
                        }
                }
                // quad layout plane[band][col/4][row][col%4]: the 32 lanes (rows) of a
                // warp store 512 contiguous bytes per instruction
                const size_t q0 = (size_t)W.y * (P.Np >> 2) + ((size_t)(n0 + col0 + 32 * h) >> 2);
                if (!(P.debug & 2)) {
#pragma unroll
                    for (int c = 0; c < 32; c += 4) {
                        const size_t off = (((q0 + (c >> 2)) * P.Mp + row) << 2);
                        *(uint4*)(P.Tw + off) = make_uint4(word[c], word[c + 1], word[c + 2], word[c + 3]);
                        int4 t = make_int4(carry[c], carry[c + 1], carry[c + 2], carry[c + 3]);
                        if (n_norm) {  // plus the carries folded out by the normalisations
                            const int4 o = *(int4*)(P.Tc + off);
                            t.x += o.x;
                            t.y += o.y;
                            t.z += o.z;
                            t.w += o.w;
                        }
                        *(int4*)(P.Tc + off) = t;
                    }
                }
            }
            fence_before();
            if (P.dbg_ts && warp == 2 && lane == 0 && it - it_begin < 4) P.dbg_ts[blockIdx.x * 32 + 8 * (it - it_begin) + 4] = clock64();
            mbar_arrive(tempty);
            tph ^= 1;
        }
    }

    fence_before();
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                     : "memory");
    }
    span_timer_exit(P.timer);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}

int make_map(CUtensorMap* m, const void* base, uint64_t inner_bytes, uint64_t rows, uint32_t box_rows) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return APB_ERR_CUDA;
    }
    cuuint64_t dims[2] = {inner_bytes, rows};
    cuuint64_t strides[1] = {inner_bytes};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed");
        return APB_ERR_CUDA;
    }
    return APB_OK;
}

}  // namespace

int slice_gemm_launch(const int8_t* Apack, const int8_t* Bpack, const SliceGemmParams& P, int n_groups,
                      cudaStream_t st) {
    CUtensorMap ma, mb;
    int rc = make_map(&ma, Apack, (uint64_t)P.Kp, (uint64_t)P.S_A * P.Mp, BM);
    if (rc) return rc;
    rc = make_map(&mb, Bpack, (uint64_t)P.Kp, (uint64_t)P.S_B * P.Np, BN);
    if (rc) return rc;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(slice_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
        attr = true;
    }
    dim3 grid((unsigned)n_groups, (unsigned)(P.Mp / BM), (unsigned)(P.Np / BN));
    const int tok = prof_begin("slice_gemm", st);
    slice_gemm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(ma, mb, P);
    prof_end(tok, st);
    count_launch();
    return cuda_check(cudaGetLastError(), "slice_gemm launch");
}

}  // namespace apb

namespace apb {

template <int BNT, int W>
static int band_launch_t(const CUtensorMap& ma, const CUtensorMap& mb, const BandGemmParams& P, int n_ctas,
                         cudaStream_t st) {
    using Cfg = BandCfg<BNT, W>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(band_gemm_kernel<BNT, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        cudaFuncSetAttribute(band3_gemm_kernel<BNT, W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        cudaFuncSetAttribute(band3_gemm_kernel<BNT, W, W == 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        cudaFuncSetAttribute(band3_gemm_kernel<BNT, W, W == 2, W == 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
        // full shared-memory carveout, so the SM keeps room for a co-resident radius block
        cudaFuncSetAttribute(band3_gemm_kernel<BNT, W, false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(band3_gemm_kernel<BNT, W, W == 2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    static const bool v2 = std::getenv("APB_BAND_V2") != nullptr;  // previous issue loop (A/B timing)
    if (v2) {
        band_gemm_kernel<BNT, W><<<n_ctas, THREADS, Cfg::SMEM, st>>>(ma, mb, P);
        return APB_OK;
    }
    // highest launch priority: the persistent CTAs (one per SM) take SMs ahead of
    // the radius products queued on the side stream
    static const int prio = [] {
        int least = 0, greatest = 0;
        cudaDeviceGetStreamPriorityRange(&least, &greatest);
        return std::getenv("APB_NO_PRIO") ? least : greatest;
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)n_ctas);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = Cfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = prio;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (W == 2 && P.raw && P.n_bands > 0) cudaLaunchKernelEx(&cfg, band3_gemm_kernel<BNT, W, W == 2, W == 2>, ma, mb, P);  // K split
    else if (W == 2 && P.raw) cudaLaunchKernelEx(&cfg, band3_gemm_kernel<BNT, W, W == 2>, ma, mb, P);
    else cudaLaunchKernelEx(&cfg, band3_gemm_kernel<BNT, W, false>, ma, mb, P);
    return APB_OK;
}

unsigned long long* gemm_timer() {
    static unsigned long long* t = [] {
        unsigned long long* p = nullptr;
        cudaMalloc(&p, 8 * sizeof(unsigned long long));
        const unsigned long long init[8] = {0, 0, ~0ull, 0, 0, 0, 0, 0};
        cudaMemcpy(p, init, sizeof init, cudaMemcpyHostToDevice);
        return p;
    }();
    return t;
}

static int g_last_cfg[4] = {0, 0, 0, 0};

int band_gemm_launch(const int8_t* Apack, const int8_t* Bpack, const BandGemmParams& Pin, int n_ctas,
                     cudaStream_t st) {
    BandGemmParams P = Pin;
    g_last_cfg[0] = P.bn;
    g_last_cfg[1] = P.band_w;
    g_last_cfg[2] = P.raw;
    g_last_cfg[3] = P.n_bands > 0 ? (P.n_kb + P.kb_per - 1) / P.kb_per : 1;
    if (!P.timer) P.timer = gemm_timer();
    CUtensorMap ma, mb;
    int rc = make_map(&ma, Apack, (uint64_t)P.Kp, (uint64_t)P.S_A * P.Mp, BM);
    if (rc) return rc;
    rc = make_map(&mb, Bpack, (uint64_t)P.Kp, (uint64_t)P.S_B * P.Np, (uint32_t)P.bn);
    if (rc) return rc;
    const int tok = prof_begin("slice_gemm", st);
    if (P.bn == 256) band_launch_t<256, 2>(ma, mb, P, n_ctas, st);
    else if (P.band_w == 2) band_launch_t<128, 2>(ma, mb, P, n_ctas, st);  // raw mode, small products
    else band_launch_t<128, 4>(ma, mb, P, n_ctas, st);
    prof_end(tok, st);
    count_launch();
    return cuda_check(cudaGetLastError(), "band_gemm launch");
}

}  // namespace apb

extern "C" {

// span timer of the band GEMM: total device time (ns, %globaltimer, first CTA
// start to last CTA end) and launch count since the last reset; graph-safe
int apb_gemm_timer_read(uint64_t* total_ns, uint64_t* launches) {
    unsigned long long h[2] = {0, 0};
    if (cudaMemcpy(h, apb::gemm_timer(), sizeof h, cudaMemcpyDeviceToHost) != cudaSuccess) return APB_ERR_CUDA;
    if (total_ns) *total_ns = h[0];
    if (launches) *launches = h[1];
    return APB_OK;
}

int apb_gemm_last_config(int* tile_n, int* band_w, int* raw, int* ksplit) {
    if (tile_n) *tile_n = apb::g_last_cfg[0];
    if (band_w) *band_w = apb::g_last_cfg[1];
    if (raw) *raw = apb::g_last_cfg[2];
    if (ksplit) *ksplit = apb::g_last_cfg[3];
    return APB_OK;
}

int apb_gemm_timer_reset(void) {
    const unsigned long long init[5] = {0, 0, ~0ull, 0, 0};
    return cudaMemcpy(apb::gemm_timer(), init, sizeof init, cudaMemcpyHostToDevice) == cudaSuccess ? APB_OK
                                                                                                  : APB_ERR_CUDA;
}

}  // extern "C"
