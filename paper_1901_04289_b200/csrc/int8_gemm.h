// int8_gemm.h - interface of the tcgen05 slice GEMM (int8_gemm.cu)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace apb {

constexpr int kSliceTile = 128;  // BM = BN
constexpr int kSliceBK = 128;    // K padding granule (bytes)

struct SliceGemmParams {
    int S_A, S_B;          // digit slices of A and B
    int Mp, Np, Kp;        // padded dims (multiples of 128)
    int n_kb;              // Kp / 128
    const int4* units;     // (d, s_lo, s_hi, flags: 1 first-of-d, 2 last-of-d)
    const int* group_unit_begin;  // [n_groups + 1]
    const int* group_d1;          // [n_groups] one past the last diagonal of the group
    uint32_t* Tw;          // [ceil(ND/4)][Mp][Np] packed result bytes
    int32_t* Tc;           // [n_groups][Mp][Np] final carry of each group
};

// band variant: 4 diagonals per pass, persistent CTAs over (tile, band) items
struct BandGemmParams {
    int S_A, S_B, Mp, Np, Kp, n_kb, ND;
    int bn, band_w;           // (128, 4) or (256, 2): output tile width / diagonals per item
    // K blocks between in-place normalisations of the TMEM accumulators (0 = none):
    // needed when pairs * K * 2^14 could reach 2^31 (high precision, long K)
    int kb_norm = 0;
    int n_tiles_n;            // Np / 128
    const int2* items;        // (tile = mt * n_tiles_n + nt, band)
    const int* cta_begin;     // [n_ctas + 1] item ranges per CTA
    uint32_t* Tw;             // [n_bands][Mp][Np] result bytes of diagonals 4b..4b+3
    int32_t* Tc;              // [n_bands][Mp][Np] carry out of band b
    // raw epilogue (no normalisations only): 1: Tw[band] = diagonal 2b, Tc[band] = diagonal 2b+1 as
    // the int32 accumulators themselves; 2 (when |D0 + 256 D1| < 2^39): Tw[band] = the low word of
    // D0 + 256 D1 and Tc, as a byte plane [band][entry], its bits 32..39; recombine16 does the
    // carry arithmetic (R.raw)
    int raw = 0;
    // raw mode only: K split.  item.y = band | ks << 16; split ks covers K blocks
    // [ks * kb_per, min(n_kb, (ks + 1) * kb_per)) and writes its own planes (index band +
    // n_bands * ks); the recombine adds the splits' accumulators
    int n_bands = 0, kb_per = 1 << 30;
    int debug = 0;            // timing experiments only: 1 skip TMA refills, 2 skip epilogue stores
    long long* dbg_ts = nullptr;  // optional per-CTA clock64 trace (timing experiments)
    unsigned long long* timer = nullptr;  // device span timer (gemm_timer_*): [sum ns, launches, start, done, end]
    // speculative launch (before the host has planned): the planner's window
    // heights (maxw_a, maxw_b) on the device; the kernel stands down unless they
    // give exactly S_A and S_B slices
    const long long* spec_maxw = nullptr;
};

// device-side span timer of the band GEMM (first CTA start to last CTA end,
// %globaltimer ns), accumulated per launch -- works inside captured graphs
unsigned long long* gemm_timer();

int band_gemm_launch(const int8_t* Apack, const int8_t* Bpack, const BandGemmParams& P, int n_ctas,
                     cudaStream_t st);

int slice_gemm_launch(const int8_t* Apack, const int8_t* Bpack, const SliceGemmParams& P, int n_groups,
                      cudaStream_t st);

}  // namespace apb
