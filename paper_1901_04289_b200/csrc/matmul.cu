// matmul.cu - ball matrix multiplication on the B200 (reference src/matmul.cpp,
// paths relative to /root/reference/proj).
//
//   matmul_auto / block / classical driver        src/matmul.cpp:442-531
//   K3  scan + plan: entry_precision, per-row / per-column bit windows, the
//       single-block test and the device greedy split    :47-52, 74-161
//   K4  scale_pack: scaled integers mid * 2^(e_i) -> balanced int8 digits in
//       slice-major, K-contiguous planes for TMA          :163-203, bigint.cpp:178-185
//   K5  slice_gemm (int8_gemm.cu): exact integer product on tcgen05
//   K6  recombine: bytes + carries -> exact integer -> * 2^(-e_i-f_j) -> ball_add
//       into C (a single block is one apfloat_round)      :476-496, bigint.cpp:187-191
//   K7  radius: |A| R_B + R_A (|B| + R_B) as scaled binary64 sums in the
//       reference's exact order (RN, no FMA, 1024-term chunks, (1+2^-29)
//       inflation), so the radius is bit-identical        :368-438, 498-513
//   K8  complex: four real products + ball add/sub       :533-548
//
// Host synchronisation: one small device->host read after the scan (the plan
// decides slice counts and block structure, as the reference's planner does).

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <functional>
#include <map>
#include <vector>

#include <cuda_runtime.h>

#include "apb.h"
#include "apb_common.cuh"
#include "apb_internal.h"
#include "int8_gemm.h"

namespace apb {

apb_matmul_stats& stats();

namespace {

struct ScanSummary {
    int special_a, special_b;
    long long prec_a, prec_b;   // entry_precision
    long long maxw_a, maxw_b;   // max row / column window width over the scanned range
    long long mw[8];            // block_matmul: radius window widths / nonzero counts (mw1, mw2)
    int rad_centred;            // 1: an operand exponent exceeds +-kRadUncentred (centred planes needed)
    int _pad;
};

// bit width of a finite nonzero midpoint stored in L top-aligned slots
APB_DEV int64_t slot_bitwidth(const uint64_t* m, int L) {
    int z = 0;
    while (z < L - 1 && m[z] == 0) z++;
    return 64 * (int64_t)L - (64 * (int64_t)z + (int64_t)ctz64(m[z]));
}

APB_DEV bool ball_special(const BallsView& a, int64_t e) {
    const int k = a.kind[e] & APB_KIND_MASK;
    return (k != APB_ZERO && k != APB_FINITE) || a.rad_man[e] == APB_RAD_INF;
}

// window (top, bottom) of a finite nonzero midpoint (ball_window, src/matmul.cpp:116-121)
APB_DEV bool mid_window(const BallsView& a, int64_t e, int64_t& top, int64_t& bot) {
    if ((a.kind[e] & APB_KIND_MASK) != APB_FINITE) return false;
    top = a.exp[e];
    bot = top - slot_bitwidth(a.mant + e * (int64_t)a.L, a.L);
    return true;
}

// ---------------------------------------------------------------- K3 scan

// warp per row of A: window over columns [lo,hi), specials, entry precision
__global__ void scan_rows_kernel(BallsView A, int64_t M, int64_t K, int64_t lo, int64_t hi,
                                 int64_t* rtop, int64_t* rbot, ScanSummary* sum) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= M) return;
    int64_t top = INT64_MIN, bot = INT64_MAX, prec = 0;
    int special = 0;
    for (int64_t k = lo + lane; k < hi; k += 32) {
        const int64_t e = i * K + k;
        special |= ball_special(A, e);
        int64_t t, b;
        if (mid_window(A, e, t, b)) {
            top = t > top ? t : top;
            bot = b < bot ? b : bot;
            prec = (t - b) > prec ? (t - b) : prec;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        int64_t t2 = __shfl_xor_sync(0xffffffffu, top, o);
        int64_t b2 = __shfl_xor_sync(0xffffffffu, bot, o);
        int64_t p2 = __shfl_xor_sync(0xffffffffu, prec, o);
        top = t2 > top ? t2 : top;
        bot = b2 < bot ? b2 : bot;
        prec = p2 > prec ? p2 : prec;
    }
    special = __any_sync(0xffffffffu, special);
    if (lane == 0) {
        rtop[i] = top;
        rbot[i] = bot;
        if (special) atomicOr(&sum->special_a, 1);
        atomicMax(&sum->prec_a, (long long)prec);
        if (top != INT64_MIN) atomicMax(&sum->maxw_a, (long long)(top - bot));
    }
}

// column windows of B over rows [lo,hi): grid (column tiles, row chunks),
// per-column int64 atomics; col_width_kernel finishes the widths
constexpr int COL_CHUNK = 16;

__global__ void init_minmax_kernel(int64_t* top, int64_t* bot, int64_t n) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) {
        top[j] = INT64_MIN;
        bot[j] = INT64_MAX;
    }
}

__global__ void scan_cols_kernel(BallsView B, int64_t K, int64_t N, int64_t lo, int64_t hi,
                                 int64_t* ctop, int64_t* cbot, ScanSummary* sum) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k0 = lo + (int64_t)blockIdx.y * COL_CHUNK;
    const int64_t k1 = k0 + COL_CHUNK < hi ? k0 + COL_CHUNK : hi;
    int64_t top = INT64_MIN, bot = INT64_MAX, prec = 0;
    int special = 0;
    if (j < N) {
        for (int64_t k = k0; k < k1; k++) {
            const int64_t e = k * N + j;
            special |= ball_special(B, e);
            int64_t t, b;
            if (mid_window(B, e, t, b)) {
                top = t > top ? t : top;
                bot = b < bot ? b : bot;
                prec = (t - b) > prec ? (t - b) : prec;
            }
        }
        if (top != INT64_MIN) {
            atomicMax((long long*)&ctop[j], (long long)top);
            atomicMin((long long*)&cbot[j], (long long)bot);
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        int64_t p2 = __shfl_xor_sync(0xffffffffu, prec, o);
        prec = p2 > prec ? p2 : prec;
    }
    special = __any_sync(0xffffffffu, special);
    if ((threadIdx.x & 31) == 0) {
        if (special) atomicOr(&sum->special_b, 1);
        if (prec) atomicMax(&sum->prec_b, (long long)prec);
    }
}

__global__ void col_width_kernel(const int64_t* ctop, const int64_t* cbot, int64_t N, long long* maxw) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long w = 0;
    if (j < N && ctop[j] != INT64_MIN) w = (long long)(ctop[j] - cbot[j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        long long w2 = __shfl_xor_sync(0xffffffffu, w, o);
        w = w2 > w ? w2 : w;
    }
    if ((threadIdx.x & 31) == 0 && w) atomicMax(maxw, w);
}

// ----------------------------------------------------- K3 greedy (device)
// greedy_split (src/matmul.cpp:74-114) over per-entry windows wA[i*K+k],
// wB[j*K+k] (top == INT64_MIN marks an empty entry); one CTA, sequential in k.
__global__ void greedy_kernel(const longlong2* wA, const longlong2* wB, int64_t K, int64_t M,
                              int64_t N, int64_t h, int64_t* out, int* nout) {
    extern __shared__ longlong2 win[];  // M rows then N cols: (top, bot)
    __shared__ int s_ok;
    const int64_t R = M + N;
    for (int64_t r = threadIdx.x; r < R; r += blockDim.x) win[r] = make_longlong2(INT64_MIN, INT64_MAX);
    int64_t lo = 0, k = 0;
    int cnt = 0;
    __syncthreads();
    while (lo < K) {
        if (threadIdx.x == 0) s_ok = 1;
        __syncthreads();
        if (k != lo) {
            bool ok = true;
            for (int64_t r = threadIdx.x; r < R && ok; r += blockDim.x) {
                longlong2 e = r < M ? wA[r * K + k] : wB[(r - M) * K + k];
                if (e.x == INT64_MIN) continue;
                longlong2 w = win[r];
                int64_t wd = w.x == INT64_MIN ? e.x - e.y : max(w.x, e.x) - min(w.y, e.y);
                if (wd > h) ok = false;
            }
            if (!ok) s_ok = 0;
        }
        __syncthreads();
        const bool ok = s_ok != 0;
        if (ok) {
            for (int64_t r = threadIdx.x; r < R; r += blockDim.x) {
                longlong2 e = r < M ? wA[r * K + k] : wB[(r - M) * K + k];
                if (e.x == INT64_MIN) continue;
                longlong2 w = win[r];
                win[r] = w.x == INT64_MIN ? e : make_longlong2(max(w.x, e.x), min(w.y, e.y));
            }
            if (++k == K) {
                if (threadIdx.x == 0) {
                    out[2 * cnt] = lo;
                    out[2 * cnt + 1] = k;
                }
                cnt++;
                lo = k;
            }
        } else {
            if (threadIdx.x == 0) {
                out[2 * cnt] = lo;
                out[2 * cnt + 1] = k;
            }
            cnt++;
            lo = k;
            for (int64_t r = threadIdx.x; r < R; r += blockDim.x) win[r] = make_longlong2(INT64_MIN, INT64_MAX);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *nout = cnt;
}

// per-entry midpoint windows, transposed to [row][k] / [col][k]
__global__ void entry_windows_kernel(BallsView A, BallsView B, int64_t M, int64_t K, int64_t N,
                                     longlong2* wA, longlong2* wB) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < M * K) {
        int64_t tp, bt;
        wA[t] = mid_window(A, t, tp, bt) ? make_longlong2(tp, bt) : make_longlong2(INT64_MIN, INT64_MAX);
    } else if (t < M * K + K * N) {
        const int64_t u = t - M * K;  // u = j*K + k
        const int64_t j = u / K, k = u % K;
        int64_t tp, bt;
        wB[u] = mid_window(B, k * N + j, tp, bt) ? make_longlong2(tp, bt) : make_longlong2(INT64_MIN, INT64_MAX);
    }
}

// ------------------------------------------------------------- K4 pack
// Digit state of one scaled entry, streamed 8 digits at a time: the
// magnitude bits come from two neighbouring mantissa limbs (funnel shift),
// two's complement negation and balanced recoding run byte-serially.
struct DigitStream {
    const uint64_t* m;  // L top-aligned limbs (global, L1-cached)
    int L;
    int64_t sh;         // value = X_L * 2^sh
    uint32_t negc, rc;
    bool neg, live;
};

APB_DEV void ds_init(DigitStream& d, const BallsView& X, int64_t e, bool valid, int64_t scale) {
    d.live = valid && (X.kind[e] & APB_KIND_MASK) == APB_FINITE;
    d.negc = 1;
    d.rc = 0;
    d.L = X.L;
    d.m = X.mant + e * (int64_t)X.L;
    d.neg = d.live && (X.kind[e] & APB_SIGN) != 0;
    d.sh = d.live ? X.exp[e] - 64 * (int64_t)X.L + scale : 0;
}

// 64 bits of X_L starting at bit position q (zeros outside)
APB_DEV uint64_t ds_word(const DigitStream& d, int64_t q) {
    if (q >= 64 * (int64_t)d.L || q <= -64) return 0;
    if (q < 0) return __ldg(d.m) << (-q);
    const int li = (int)(q >> 6), bo = (int)(q & 63);
    uint64_t v = __ldg(d.m + li) >> bo;
    if (bo && li + 1 < d.L) v |= __ldg(d.m + li + 1) << (64 - bo);
    return v;
}

// 8 balanced digits (bytes 8c .. 8c+7) from the 64 source bits w, packed little-endian
APB_DEV uint64_t ds_digits8(DigitStream& d, uint64_t w) {
    if (!d.live) return 0;
    uint64_t out = 0;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        uint32_t byte = (uint32_t)(w >> (8 * b)) & 255u;
        if (d.neg) {
            const uint32_t t = (255u - byte) + d.negc;
            byte = t & 255u;
            d.negc = t >> 8;
        }
        const uint32_t v = byte + d.rc;
        d.rc = v >= 128 ? 1u : 0u;
        out |= (uint64_t)(v & 255u) << (8 * b);  // (v - 256) as a byte == v & 255
    }
    return out;
}

// Pack 4 consecutive inner indices per thread: plane[s][row][kk..kk+3] (one
// 32-bit store per plane).  IS_B: entry (lo+kk, row) of B with column scale.
template <bool IS_B>
__global__ void __launch_bounds__(256) pack_kernel(BallsView X, int64_t rows, int64_t ld, int64_t lo,
                                                   int64_t hi, const int64_t* top, const int64_t* bot, int S,
                                                   int Rp, int Kp, int8_t* out, int64_t* scale_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t kq = Kp / 4;
    if (t >= (int64_t)Rp * kq) return;
    const int64_t r = t / kq, kk0 = 4 * (t % kq);
    int64_t sc = 0;
    if (r < rows) sc = top[r] == INT64_MIN ? 0 : -bot[r];
    if (r < rows && kk0 == 0) scale_out[r] = sc;
    DigitStream ds[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t kk = kk0 + q;
        const bool valid = r < rows && kk < hi - lo;
        const int64_t e = valid ? (IS_B ? (lo + kk) * ld + r : r * ld + lo + kk) : 0;
        ds_init(ds[q], X, e, valid, sc);
    }
    const size_t plane = (size_t)Rp * Kp;
    uint32_t* dst = (uint32_t*)(out + (size_t)r * Kp + kk0);
    const int nch = (S + 7) / 8;
    for (int c0 = 0; c0 < nch; c0 += 4) {
        uint64_t src[4][4];  // [chunk][entry] source words, all loads issued up front
#pragma unroll
        for (int cc = 0; cc < 4; cc++)
#pragma unroll
            for (int q = 0; q < 4; q++)
                src[cc][q] = (c0 + cc < nch && ds[q].live) ? ds_word(ds[q], 64 * (int64_t)(c0 + cc) - ds[q].sh) : 0;
#pragma unroll
        for (int cc = 0; cc < 4; cc++) {
            const int c = c0 + cc;
            if (c >= nch) break;
            uint64_t w[4];
#pragma unroll
            for (int q = 0; q < 4; q++) w[q] = ds_digits8(ds[q], src[cc][q]);
#pragma unroll
            for (int b = 0; b < 8; b++) {
                const int s = 8 * c + b;
                if (s >= S) break;
                const uint32_t word = ((uint32_t)(w[0] >> (8 * b)) & 255u) | (((uint32_t)(w[1] >> (8 * b)) & 255u) << 8) |
                                      (((uint32_t)(w[2] >> (8 * b)) & 255u) << 16) |
                                      (((uint32_t)(w[3] >> (8 * b)) & 255u) << 24);
                dst[(size_t)s * plane / 4] = word;
            }
        }
    }
}


// ---- pack v2.  Balanced digits by one multi-word addition: with X the S-byte
// two's complement of the scaled entry, Y = X + 0x8080...80 makes the carry out
// of every byte exactly the balanced-recoding carry (byte + c >= 128), and
// Y ^ 0x8080...80 are the digit bytes -- the same bytes as the byte-serial
// recoding of ds_digits8, in a handful of 64-bit ops per 8 digits.
// Up to NCW 64-bit digit words (S <= 8 NCW); magnitude bits come straight
// from the entry's limbs (loaded once, up front).
template <int NCW>
APB_DEV void digit_words(const BallsView& X, int64_t e, bool valid, int64_t scale, uint64_t (&d)[NCW]) {
    const uint8_t kd = valid ? X.kind[e] : (uint8_t)APB_ZERO;
    const bool live = (kd & APB_KIND_MASK) == APB_FINITE;
    const bool neg = live && (kd & APB_SIGN);
    const int L = X.L;
    const int64_t sh = live ? X.exp[e] - 64 * (int64_t)L + scale : 0;
    // word c = magnitude bits [64c, 64c + 64) = limbs li = c + lq (shifted right by bo)
    const int64_t lq = (-sh) >> 6;  // floor
    const int bo = (int)((-sh) & 63);
    const uint64_t* m = X.mant + e * (int64_t)L;
    uint64_t g[NCW + 1];
#pragma unroll
    for (int c = 0; c <= NCW; c++) {
        const int64_t li = c + lq;
        g[c] = (live && li >= 0 && li < L) ? __ldg(m + li) : 0ull;
    }
    uint64_t cy = neg ? 1ull : 0ull;
    constexpr uint64_t K80 = 0x8080808080808080ull;
#pragma unroll
    for (int c = 0; c < NCW; c++) {
        uint64_t w = bo ? (g[c] >> bo) | (g[c + 1] << (64 - bo)) : g[c];
        if (neg) w = ~w;
        const uint64_t s1 = w + K80;
        const uint64_t c1 = s1 < w ? 1ull : 0ull;
        const uint64_t s2 = s1 + cy;
        cy = c1 | (s2 < s1 ? 1ull : 0ull);
        d[c] = s2 ^ K80;
    }
}

// window (top, bottom) of line `line` from the scan's chunk partials P[f][c][line]
APB_DEV void partial_window(const int64_t* P, int nc, int64_t nlines, int64_t line, int64_t& top, int64_t& bot) {
    top = INT64_MIN;
    bot = INT64_MAX;
    const int64_t stride = (int64_t)nc * nlines;
    for (int c = 0; c < nc; c++) {
        const int64_t t = P[(int64_t)c * nlines + line], b = P[stride + (int64_t)c * nlines + line];
        top = t > top ? t : top;
        bot = b < bot ? b : bot;
    }
}

// A side: thread per entry (row r, inner kk), plane[s][r][kk] byte stores --
// a warp writes one 32-byte segment per plane
template <int NCW>
APB_DEV void pack_a_v2_body(const BallsView& X, int64_t rows, int64_t ld, int64_t lo, int64_t hi,
                            const int64_t* top, const int64_t* bot, int S, int Rp, int Kp, int8_t* out,
                            int64_t* scale_out, const long long* maxw_dev, int64_t blk,
                            const int64_t* part = nullptr, int nc = 0, int planes = 0) {
    if (part) {  // early pack: the planes the caller asks for, else all of the template
        S = planes > 0 && planes <= 8 * NCW ? planes : 8 * NCW;
    } else if (maxw_dev) {  // speculative launch: slice count from the scan, before the host knows it
        S = (int)((*maxw_dev + 2 + 7) / 8);
        if (S > 8 * NCW) return;
    }
    const int64_t t = blk * blockDim.x + threadIdx.x;
    if (t >= (int64_t)Rp * Kp) return;
    const int64_t r = t / Kp, kk = t % Kp;
    int64_t sc = 0;
    if (r < rows && part) {
        int64_t tp, bt;
        partial_window(part, nc, rows, r, tp, bt);
        sc = tp == INT64_MIN ? 0 : -bt;
    } else if (r < rows) sc = top[r] == INT64_MIN ? 0 : -bot[r];
    if (r < rows && kk == 0) scale_out[r] = sc;
    const bool valid = r < rows && kk < hi - lo;
    uint64_t d[NCW];
    digit_words<NCW>(X, valid ? r * ld + lo + kk : 0, valid, sc, d);
    const size_t plane = (size_t)Rp * Kp;
    int8_t* dst = out + (size_t)r * Kp + kk;
#pragma unroll
    for (int q = 0; q < 8 * NCW; q++) {
        if (q < S) dst[(size_t)q * plane] = (int8_t)(uint8_t)(d[q >> 3] >> (8 * (q & 7)));
    }
}

// A side, four consecutive inner indices per thread: the digit bytes of the four entries are merged
// with byte permutes and leave as one 4-byte store per plane (a warp writes 128 contiguous bytes per
// plane instead of 32: a quarter of the store instructions of pack_a_v2_body).  blk counts blocks of
// 256 threads over Rp * Kp / 4 thread slots.
template <int NCW>
APB_DEV void pack_a_v4_body(const BallsView& X, int64_t rows, int64_t ld, int64_t lo, int64_t hi,
                            const int64_t* top, const int64_t* bot, int S, int Rp, int Kp, int8_t* out,
                            int64_t* scale_out, const long long* maxw_dev, int64_t blk,
                            const int64_t* part = nullptr, int nc = 0, int planes = 0) {
    if (part) {
        S = planes > 0 && planes <= 8 * NCW ? planes : 8 * NCW;
    } else if (maxw_dev) {
        S = (int)((*maxw_dev + 2 + 7) / 8);
        if (S > 8 * NCW) return;
    }
    const int64_t t = blk * blockDim.x + threadIdx.x;
    const int64_t K4 = Kp >> 2;
    if (t >= (int64_t)Rp * K4) return;
    const int64_t r = t / K4, kk = 4 * (t % K4);
    int64_t sc = 0;
    if (r < rows && part) {
        int64_t tp, bt;
        partial_window(part, nc, rows, r, tp, bt);
        sc = tp == INT64_MIN ? 0 : -bt;
    } else if (r < rows) sc = top[r] == INT64_MIN ? 0 : -bot[r];
    if (r < rows && kk == 0) scale_out[r] = sc;
    uint64_t d[4][NCW];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const bool valid = r < rows && kk + q < hi - lo;
        digit_words<NCW>(X, valid ? r * ld + lo + kk + q : 0, valid, sc, d[q]);
    }
    const size_t plane = (size_t)Rp * Kp;
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + (size_t)r * Kp + kk);
#pragma unroll
    for (int c = 0; c < NCW; c++) {
        if (8 * c >= S) break;
        const uint64_t w0 = d[0][c], w1 = d[1][c], w2 = d[2][c], w3 = d[3][c];
        // byte b of (w0, w1, w2, w3) -> the word of digit 8 c + b (as pack_b_v2_body)
        const uint32_t lo01 = __byte_perm((uint32_t)w0, (uint32_t)w1, 0x5140);
        const uint32_t lo23 = __byte_perm((uint32_t)w2, (uint32_t)w3, 0x5140);
        const uint32_t hi01 = __byte_perm((uint32_t)w0, (uint32_t)w1, 0x7362);
        const uint32_t hi23 = __byte_perm((uint32_t)w2, (uint32_t)w3, 0x7362);
        const uint32_t lo01b = __byte_perm((uint32_t)(w0 >> 32), (uint32_t)(w1 >> 32), 0x5140);
        const uint32_t lo23b = __byte_perm((uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32), 0x5140);
        const uint32_t hi01b = __byte_perm((uint32_t)(w0 >> 32), (uint32_t)(w1 >> 32), 0x7362);
        const uint32_t hi23b = __byte_perm((uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32), 0x7362);
        const uint32_t dg[8] = {__byte_perm(lo01, lo23, 0x5410),   __byte_perm(lo01, lo23, 0x7632),
                                __byte_perm(hi01, hi23, 0x5410),   __byte_perm(hi01, hi23, 0x7632),
                                __byte_perm(lo01b, lo23b, 0x5410), __byte_perm(lo01b, lo23b, 0x7632),
                                __byte_perm(hi01b, hi23b, 0x5410), __byte_perm(hi01b, hi23b, 0x7632)};
#pragma unroll
        for (int b = 0; b < 8; b++)
            if (8 * c + b < S) dst[((size_t)(8 * c + b) * plane) >> 2] = dg[b];
    }
}

template <int NCW>
__global__ void __launch_bounds__(256) pack_a_v2_kernel(BallsView X, int64_t rows, int64_t ld, int64_t lo, int64_t hi,
                                                        const int64_t* top, const int64_t* bot, int S, int Rp, int Kp,
                                                        int8_t* out, int64_t* scale_out,
                                                        const long long* maxw_dev = nullptr) {
    pack_a_v2_body<NCW>(X, rows, ld, lo, hi, top, bot, S, Rp, Kp, out, scale_out, maxw_dev, blockIdx.x);
}

// B side: 32 columns x 32 inner indices per 256 threads (4 consecutive kk per
// thread, reads coalesced over columns j); digit bytes of 4 entries are merged
// with byte permutes and transposed through shared memory so plane rows (fixed
// j, contiguous kk) leave as 32-byte segments.
template <int NCW>
APB_DEV void pack_b_v2_body(const BallsView& X, int64_t N, int64_t lo, int64_t hi, const int64_t* top,
                            const int64_t* bot, int S, int Np, int Kp, int8_t* out, int64_t* scale_out,
                            const long long* maxw_dev, int64_t bx, int64_t by, const int64_t* part = nullptr,
                            int nc = 0, int planes = 0) {
    if (part) {
        S = planes > 0 && planes <= 8 * NCW ? planes : 8 * NCW;
    } else if (maxw_dev) {
        S = (int)((*maxw_dev + 2 + 7) / 8);
        if (S > 8 * NCW) return;
    }
    __shared__ uint32_t tile[8][32][9];  // [digit in chunk][j][kk word], padded
    const int jl = threadIdx.x & 31, kq = threadIdx.x >> 5;
    const int64_t j = bx * 32 + jl;
    const int64_t kk0 = by * 32 + 4 * kq;
    int64_t sc = 0;
    if (j < N && part) {
        int64_t tp, bt;
        partial_window(part, nc, N, j, tp, bt);
        sc = tp == INT64_MIN ? 0 : -bt;
    } else if (j < N) sc = top[j] == INT64_MIN ? 0 : -bot[j];
    if (j < N && by == 0 && kq == 0) scale_out[j] = sc;
    uint64_t d[4][NCW];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t kk = kk0 + q;
        const bool valid = j < N && kk < hi - lo;
        digit_words<NCW>(X, valid ? (lo + kk) * N + j : 0, valid, sc, d[q]);
    }
    const size_t plane = (size_t)Np * Kp;
#pragma unroll
    for (int c = 0; c < NCW; c++) {
        if (8 * c >= S) break;
        const uint64_t w0 = d[0][c], w1 = d[1][c], w2 = d[2][c], w3 = d[3][c];
        // byte b of (w0, w1, w2, w3) -> the word of digit 8c + b
        const uint32_t lo01 = __byte_perm((uint32_t)w0, (uint32_t)w1, 0x5140);  // w0.b0 w1.b0 w0.b1 w1.b1
        const uint32_t lo23 = __byte_perm((uint32_t)w2, (uint32_t)w3, 0x5140);
        const uint32_t hi01 = __byte_perm((uint32_t)w0, (uint32_t)w1, 0x7362);  // w0.b2 w1.b2 w0.b3 w1.b3
        const uint32_t hi23 = __byte_perm((uint32_t)w2, (uint32_t)w3, 0x7362);
        const uint32_t lo01b = __byte_perm((uint32_t)(w0 >> 32), (uint32_t)(w1 >> 32), 0x5140);
        const uint32_t lo23b = __byte_perm((uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32), 0x5140);
        const uint32_t hi01b = __byte_perm((uint32_t)(w0 >> 32), (uint32_t)(w1 >> 32), 0x7362);
        const uint32_t hi23b = __byte_perm((uint32_t)(w2 >> 32), (uint32_t)(w3 >> 32), 0x7362);
        tile[0][jl][kq] = __byte_perm(lo01, lo23, 0x5410);
        tile[1][jl][kq] = __byte_perm(lo01, lo23, 0x7632);
        tile[2][jl][kq] = __byte_perm(hi01, hi23, 0x5410);
        tile[3][jl][kq] = __byte_perm(hi01, hi23, 0x7632);
        tile[4][jl][kq] = __byte_perm(lo01b, lo23b, 0x5410);
        tile[5][jl][kq] = __byte_perm(lo01b, lo23b, 0x7632);
        tile[6][jl][kq] = __byte_perm(hi01b, hi23b, 0x5410);
        tile[7][jl][kq] = __byte_perm(hi01b, hi23b, 0x7632);
        __syncthreads();
        // 8 digits x 32 rows x 8 words: thread -> (digit b, row r, word m)
#pragma unroll
        for (int it = 0; it < 8; it++) {
            const int idx = it * 256 + threadIdx.x;
            const int m = idx & 7, r = (idx >> 3) & 31, b = idx >> 8;
            const int sdig = 8 * c + b;
            const int64_t jj = bx * 32 + r;
            if (sdig < S && jj < Np)
                *(uint32_t*)(out + (size_t)sdig * plane + (size_t)jj * Kp + (size_t)by * 32 + 4 * m) =
                    tile[b][r][m];
        }
        __syncthreads();
    }
}

template <int NCW>
__global__ void __launch_bounds__(256) pack_b_v2_kernel(BallsView X, int64_t N, int64_t lo, int64_t hi,
                                                        const int64_t* top, const int64_t* bot, int S, int Np, int Kp,
                                                        int8_t* out, int64_t* scale_out,
                                                        const long long* maxw_dev = nullptr) {
    pack_b_v2_body<NCW>(X, N, lo, hi, top, bot, S, Np, Kp, out, scale_out, maxw_dev, blockIdx.x, blockIdx.y);
}

// speculative single-block pack of both operands in one launch: blocks [0, ga)
// pack A (thread per entry), the rest pack B (32 x 32 tiles, gbx per row of tiles)
struct PackAB {
    BallsView a, b;
    int64_t M, K, N;
    const int64_t *rtop, *rbot, *ctop, *cbot;
    int Mp, Np, Kp;
    int8_t *Ap, *Bp;
    int64_t *esc, *fsc;
    const long long *mwa, *mwb;
    int64_t ga, gbx;
    // early pack (right after the scan, beside the finish kernel): the line windows come from the
    // scan's chunk partials (fields 0 / 1 = top / bottom, cA chunks per row, cB per column) and
    // every template plane is written (the slice counts are the finish kernel's to know)
    const int64_t *pa = nullptr, *pb = nullptr;
    int cA = 0, cB = 0;
    int planes_a = 0, planes_b = 0;  // early pack: planes to write (0 = all 8 NCW of the template)
    int a4 = 0;  // A side: four inner indices per thread (ga counts blocks over Mp * Kp / 4 slots)
};


template <int NCW>
#ifdef APB_PACK_MINB  // occupancy experiments (5 / 6 blocks per SM measured no faster: profiles/r2/README.md)
__global__ void __launch_bounds__(256, APB_PACK_MINB) pack_ab_v2_kernel(PackAB P) {
#else
__global__ void __launch_bounds__(256) pack_ab_v2_kernel(PackAB P) {
#endif
    griddep_wait();
    // the B blocks (4 entries per thread + a shared-memory transpose) are the long
    // ones: they take the low block indices so they are dispatched first
    const int64_t nb = P.gbx * (P.Kp / 32);
    if ((int64_t)blockIdx.x < nb) {
        const int64_t bb = blockIdx.x;
        pack_b_v2_body<NCW>(P.b, P.N, 0, P.K, P.ctop, P.cbot, 0, P.Np, P.Kp, P.Bp, P.fsc, P.mwb, bb % P.gbx,
                            bb / P.gbx, P.pb, P.cB, P.planes_b);
    } else {
        if (P.a4)
            pack_a_v4_body<NCW>(P.a, P.M, P.K, 0, P.K, P.rtop, P.rbot, 0, P.Mp, P.Kp, P.Ap, P.esc, P.mwa,
                                (int64_t)blockIdx.x - nb, P.pa, P.cA, P.planes_a);
        else
            pack_a_v2_body<NCW>(P.a, P.M, P.K, 0, P.K, P.rtop, P.rbot, 0, P.Mp, P.Kp, P.Ap, P.esc, P.mwa,
                                (int64_t)blockIdx.x - nb, P.pa, P.cA, P.planes_a);
    }
}

// B-side pack with coalesced reads: a 32 (columns j) x 32 (inner kk) tile per
// 256 threads; lanes run over consecutive j (contiguous in row-major B), the
// digits are transposed through shared memory so each plane row (fixed j,
// contiguous kk) is written with 32-byte segments.
__global__ void __launch_bounds__(256) pack_b_tiled_kernel(BallsView X, int64_t N, int64_t lo, int64_t hi,
                                                           const int64_t* top, const int64_t* bot, int S,
                                                           int Np, int Kp, int8_t* out, int64_t* scale_out) {
    __shared__ uint32_t tile[8][32][9];  // [digit in chunk][j][kk word], padded
    const int jl = threadIdx.x & 31, kq = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + jl;
    const int64_t kk0 = (int64_t)blockIdx.y * 32 + 4 * kq;
    int64_t sc = 0;
    if (j < N) sc = top[j] == INT64_MIN ? 0 : -bot[j];
    if (j < N && blockIdx.y == 0 && kq == 0) scale_out[j] = sc;
    DigitStream ds[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t kk = kk0 + q;
        const bool valid = j < N && kk < hi - lo;
        ds_init(ds[q], X, valid ? (lo + kk) * N + j : 0, valid, sc);
    }
    const size_t plane = (size_t)Np * Kp;
    const int nch = (S + 7) / 8;
    for (int c = 0; c < nch; c++) {
        uint64_t w[4];
#pragma unroll
        for (int q = 0; q < 4; q++) w[q] = ds_digits8(ds[q], ds[q].live ? ds_word(ds[q], 64 * (int64_t)c - ds[q].sh) : 0);
#pragma unroll
        for (int b = 0; b < 8; b++)
            tile[b][jl][kq] = ((uint32_t)(w[0] >> (8 * b)) & 255u) | (((uint32_t)(w[1] >> (8 * b)) & 255u) << 8) |
                              (((uint32_t)(w[2] >> (8 * b)) & 255u) << 16) | (((uint32_t)(w[3] >> (8 * b)) & 255u) << 24);
        __syncthreads();
        // 8 digits x 32 rows x 8 words: thread -> (digit b, row r, word m)
#pragma unroll
        for (int it = 0; it < 8; it++) {
            const int idx = it * 256 + threadIdx.x;
            const int m = idx & 7, r = (idx >> 3) & 31, b = idx >> 8;
            const int s = 8 * c + b;
            const int64_t jj = (int64_t)blockIdx.x * 32 + r;
            if (s < S && jj < Np)
                *(uint32_t*)(out + (size_t)s * plane + (size_t)jj * Kp + (size_t)blockIdx.y * 32 + 4 * m) = tile[b][r][m];
        }
        __syncthreads();
    }
}

// -------------------------------------------------------- K6 recombine
struct RecombineArgs {
    const uint32_t* Tw;
    const int32_t* Tc;
    const int* group_d1;
    int n_groups, nwords;
    int Mp, Np;
    int64_t M, N;
    const int64_t* escale;
    const int64_t* fscale;
    BallsOut C;
    int first;  // C is still all-zero (single block or first scaled block)
    int64_t prec;
    int64_t* int_out;  // optional: exact integer limbs (two's complement), int_limbs per entry
    int int_limbs;
    int* status;
    int quad;  // band GEMM layout: plane[(j/4)][i][j%4] (coalesced epilogue stores), else [i][j]
    int digit_bits = 32;  // bits per Tw plane digit: 8 x diagonals per word
    // raw band planes (recombine16 only): 1: Tw[b] / Tc[b] are the int32 accumulators of
    // diagonals 2b / 2b+1; 2: Tw[b] is the low word of D0 + 256 D1 and Tc a byte plane with its
    // bits 32..39 (BandGemmParams::raw); band b contributes D0 + 256 D1 at digit b
    int raw = 0;
    int nsplit = 1;  // raw mode: K splits (1 or 2), the second split's planes start at plane index nwords
    // optional fused radius combine (recombine16 only): C.rad = err (+) (r1 (+) r2), the
    // rad_combine_kernel step of src/matmul.cpp:512-513 folded into the store
    const uint32_t* r1b = nullptr;
    const int64_t* r1f = nullptr;
    const uint32_t* r2b = nullptr;
    const int64_t* r2f = nullptr;
    // speculative launch: stand down unless the device window heights give (sa, sb) slices
    const long long* spec_maxw = nullptr;
    int spec_sa = 0, spec_sb = 0;
};

APB_DEV size_t rc_off(const RecombineArgs& R, int64_t i, int64_t j) {
    return R.quad ? (((size_t)(j >> 2) * R.Mp + (size_t)i) << 2) + (size_t)(j & 3) : (size_t)i * R.Np + (size_t)j;
}

template <int CAP>
__global__ void __launch_bounds__(128) recombine_kernel(RecombineArgs R) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= R.M * R.N) return;
    const int64_t i = t / R.N, j = t % R.N;
    const size_t plane = (size_t)R.Mp * R.Np;
    const size_t off = rc_off(R, i, j);
    // T = (bytes as unsigned) + sum_g carry_g * 256^(d1_g), two's complement in NT limbs
    const int NT = (int)(((int64_t)R.digit_bits * R.nwords + 63) / 64) + 2;
    uint64_t T[CAP];
    for (int q = 0; q < NT; q++) T[q] = 0;
    // plane w holds digit w in base 2^(8 diagonals per word): 32-bit words (4 diagonals,
    // unit / 128-wide band kernel) or 16-bit digits (2 diagonals, 256-wide band kernel)
    const int db = R.digit_bits;
    for (int w = 0; w < R.nwords; w++) {
        const int64_t bit = (int64_t)db * w;
        T[bit >> 6] |= (uint64_t)R.Tw[(size_t)w * plane + off] << (bit & 63);
    }
    // carries: c_g << (8 d1_g) collected per 64-bit limb in signed 128-bit sums (each
    // term < 2^95 in magnitude, a few per limb), then one signed carry pass over T
    __int128 cs[CAP];
    for (int q = 0; q < NT; q++) cs[q] = 0;
    for (int g = 0; g < R.n_groups; g++) {
        const int64_t c = R.Tc[(size_t)g * plane + off];
        if (c == 0) continue;
        const int64_t bit = 8 * (int64_t)R.group_d1[g];
        cs[bit >> 6] += (__int128)c << (bit & 63);
    }
    {
        __int128 cy = 0;
        for (int q = 0; q < NT; q++) {
            const __int128 v = (__int128)T[q] + cs[q] + cy;
            T[q] = (uint64_t)v;
            cy = v >> 64;  // arithmetic: the sign travels up (two's complement mod 2^(64 NT))
        }
    }
    if (R.int_out)
        for (int q = 0; q < R.int_limbs; q++)
            R.int_out[t * R.int_limbs + q] = (int64_t)(q < NT ? T[q] : ((T[NT - 1] >> 63) ? ~0ull : 0ull));
    if (!R.C.mant) return;
    const bool neg = (T[NT - 1] >> 63) != 0;
    if (neg) {
        uint64_t c = 1;
        for (int q = 0; q < NT; q++) {
            uint64_t v = ~T[q] + c;
            c = (c && v == 0);
            T[q] = v;
        }
    }
    bool zero = true;
    for (int q = 0; q < NT; q++) zero &= T[q] == 0;
    if (zero) {
        if (R.first) {  // untouched C entry stays an exact zero
            GFloat<1> z;
            z.kind = APB_ZERO;
            z.neg = 0;
            z.e = 0;
            z.n = 0;
            gf_store(R.C, t, z, mag_zero(), R.status);
        }
        return;
    }
    // apfloat_from_bigint_scaled(v, -e_i - f_j) (src/bigint.cpp:187-191)
    GFloat<CAP> v;
    const int64_t exp2 = -R.escale[i] - R.fscale[j];
    gf_normalize(v, neg ? 1 : 0, checked_add(64 * (int64_t)NT, exp2, R.status), T, NT, R.status);
    if (R.first) {
        Mag err = gf_round(v, R.prec, R.status);  // ball_add(0, v): apfloat_round
        gf_store(R.C, t, v, err, R.status);
    } else {
        GF c, vv;
        vv.kind = v.kind;
        vv.neg = v.neg;
        vv.e = v.e;
        vv.n = v.n;
        for (int q = 0; q < v.n; q++) vv.d[q] = v.d[q];
        BallsView cv{R.C.mant, R.C.exp, R.C.kind, R.C.rad_man, R.C.rad_exp, R.C.L};
        gf_load(c, cv, t);
        Mag crad = mag_load(R.C.rad_man[t], R.C.rad_exp[t]);
        Mag err = gf_add_round(c, c, vv, R.prec, R.status);  // ball_add (src/ball.cpp:15-19)
        if (c.kind == APB_NAN) {
            gf_store(R.C, t, c, mag_inf(), R.status);
        } else {
            gf_store(R.C, t, c, mag_add(crad, err), R.status);
        }
    }
}


// Register-resident recombine for the band GEMM output of a single (first)
// block: T = sum_b (word_b + carry_b 2^DB) 2^(DB b) in base-2^DB digits, then
// sign, normalize and truncate to p bits with the apfloat_round error term
// (src/apfloat.cpp:26-63, 138-162), all with compile-time array bounds.
template <int NBC, int DB>
__global__ void __launch_bounds__(128) recombine_fast_kernel(RecombineArgs R) {
    // digits of DB = 8 * (diagonals per band) bits: band b's word is digit b, its carry digit b+1
    constexpr int ND32 = NBC + 2;               // digits
    constexpr int PER = 64 / DB;                // digits per 64-bit limb
    constexpr int NL = (ND32 + PER - 1) / PER;  // 64-bit limbs
    // threads walk the quad layout: t -> (j/4, i, j%4), so plane reads are contiguous
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t jr = u & 3, i = (u >> 2) % R.M, jq = (u >> 2) / R.M;
    const int64_t j = 4 * jq + jr;
    if (jq * 4 >= R.N || j >= R.N) return;
    const int64_t t = i * R.N + j;
    const size_t plane = (size_t)R.Mp * R.Np;
    const size_t off = rc_off(R, i, j);
    const int NB = R.nwords;
    // one streaming pass over the digits, base 2^DB: digit k = word_k + carry_{k-1}
    // + the running carry; batches of RB bands are loaded before they are
    // consumed so RB * 2 loads are in flight per thread with few live registers
#ifndef APB_RC16_RB
#define APB_RC16_RB 8
#endif
    constexpr int RB = APB_RC16_RB;  // band loads in flight per thread
    uint64_t T[NL];
#pragma unroll
    for (int q = 0; q < NL; q++) T[q] = 0;
    int64_t run = 0, prev_c = 0;
    bool neg = false;
#pragma unroll
    for (int kb = 0; kb < ND32; kb += RB) {
        uint32_t w[RB];
        int32_t c[RB];
#pragma unroll
        for (int u = 0; u < RB; u++) {
            const int b = kb + u;
            w[u] = (b < NBC && b < NB) ? __ldcs(R.Tw + (size_t)b * plane + off) : 0u;
            c[u] = (b < NBC && b < NB) ? __ldcs(R.Tc + (size_t)b * plane + off) : 0;
        }
        asm volatile("" ::: "memory");  // all 2 RB loads of the batch in flight
#pragma unroll
        for (int u = 0; u < RB; u++) {
            const int k = kb + u;
            if (k < ND32) {
                const int64_t d = run + (int64_t)w[u] + prev_c;
                prev_c = c[u];
                const uint64_t dg = (uint64_t)d & ((1ull << DB) - 1);
                if (k == ND32 - 1) {
                    neg = d < 0;  // the arithmetic top digit carries the sign
                } else {
                    run = d >> DB;
                }
                T[k / PER] |= dg << (DB * (k % PER));
            }
        }
    }
    if (neg) {  // sign-fill the digits above the top one, then take the magnitude
#pragma unroll
        for (int k = ND32; k < NL * PER; k++) T[k / PER] |= ((1ull << DB) - 1) << (DB * (k % PER));
        uint64_t cc = 1;
#pragma unroll
        for (int q = 0; q < NL; q++) {
            const uint64_t v = ~T[q] + cc;
            cc = (cc && v == 0) ? 1 : 0;
            T[q] = v;
        }
    }
    // bit length B of the magnitude
    int64_t B = 0;
#pragma unroll
    for (int q = 0; q < NL; q++)
        if (T[q]) B = 64 * (int64_t)q + (int64_t)bitw64(T[q]);
    BallsOut& O = R.C;
    uint64_t* dst = O.mant + t * (int64_t)O.L;
    if (B == 0) {  // exact zero: C stays Ball::zero()
        for (int q = 0; q < O.L; q++) dst[q] = 0;
        O.exp[t] = 0;
        O.kind[t] = APB_ZERO;
        O.rad_man[t] = 0;
        O.rad_exp[t] = 0;
        return;
    }
    const int64_t exp2 = -R.escale[i] - R.fscale[j];
    int st = 0;
    const int64_t e = checked_add(exp2, B, &st);  // apfloat_from_bigint_scaled exponent
    const int64_t p = R.prec;
    const int64_t cut = B > p ? B - p : 0;        // bits [0, cut) are truncated
    // bits [pos, pos + 64) of the magnitude (0 outside), static-index selects
    auto bits64 = [&](int64_t pos) -> uint64_t {
        if (pos >= 64 * (int64_t)NL || pos <= -64) return 0;
        const int64_t li = pos >= 0 ? pos >> 6 : -1;
        const int bo = (int)(pos - 64 * li);
        uint64_t lo = 0, hi = 0;
#pragma unroll
        for (int q = 0; q < NL; q++) {
            if (q == li) lo = T[q];
            if (q == li + 1) hi = T[q];
        }
        return bo ? (lo >> bo) | (hi << (64 - bo)) : lo;
    };
    // output mantissa: bits [B - 64 (r + 1), B - 64 r) for r = 0..L-1, cleared below `cut`
    for (int r = 0; r < O.L; r++) {
        const int64_t lo_bit = B - 64 * (int64_t)(r + 1);
        uint64_t v = bits64(lo_bit);
        if (lo_bit < cut) {
            const int64_t k = cut - lo_bit;  // low k bits of v are below the cut
            v = k >= 64 ? 0 : (v & ~((1ull << k) - 1));
        }
        dst[O.L - 1 - r] = v;
    }
    O.exp[t] = e;
    O.kind[t] = (uint8_t)(APB_FINITE | (neg ? APB_SIGN : 0));
    // error of the truncation: Mag upper bound of the discarded bits
    Mag err = mag_zero();
    if (cut > 0) {
        // highest set bit below the cut
        int64_t top = -1;
#pragma unroll
        for (int q = 0; q < NL; q++) {
            uint64_t v = T[q];
            const int64_t base = 64 * (int64_t)q;
            if (base >= cut) v = 0;
            else if (cut - base < 64) v &= (1ull << (cut - base)) - 1;
            if (v) top = base + (int64_t)bitw64(v) - 1;
        }
        if (top >= 0) {
            // 64-bit window starting at the top set bit, and sticky of everything below it
            const uint64_t window = bits64(top - 63);
            bool low = (window & ((1ull << 34) - 1)) != 0;
            const int64_t below = top - 63;  // bits [0, below) not in the window
#pragma unroll
            for (int q = 0; q < NL; q++) {
                uint64_t v = T[q];
                const int64_t base = 64 * (int64_t)q;
                if (base >= below) v = 0;
                else if (below - base < 64) v &= (1ull << (below - base)) - 1;
                low |= v != 0;
            }
            uint64_t bm = window >> 34;
            if (low) bm++;
            err = mag_parts(bm, checked_add(exp2, top + 1, &st));
        }
    }
    mag_store(err, &O.rad_man[t], &O.rad_exp[t]);
    if (st) *R.status = st;
}

// Recombine for 16-bit band digits (2 diagonals per band, the default
// 128x256 tile): the digit recurrence d = run + word_k + carry_{k-1} stays in
// int32 (|carry| < 2^24, word < 2^16), the magnitude words are parked in
// shared memory (one padded row per thread) so the p-bit output window and
// the truncation error are read with dynamic word indices instead of select
// chains.  Same results as recombine_fast_kernel<*, 16>.
// V40: the planes are the 40-bit raw format (R.raw == 2): only the word and byte pointers are
// stepped (the three per-band 64-bit pointer steps were 23% of the kernel's instructions)
template <int NBC, bool SPLIT = false, bool V40 = false>
__global__ void __launch_bounds__(128) recombine16_kernel(RecombineArgs R) {
    constexpr int ND = NBC + 2;        // base-2^16 digits (band b: word digit b, carry digit b+1)
    constexpr int NW = (ND + 1) / 2;   // 32-bit magnitude words
    constexpr int STR = (NW + 3) | 1;  // smem row stride, 2 guard words; forced odd: NW + 3 is 24 / 44 for
                                       // NBC = 40 / 80, and an even stride put the 32 rows of a warp on 4 banks
                                       // (ncu: 6.7 extra wavefronts per shared load)
    __shared__ uint32_t sm[128 * STR];
    griddep_wait();  // (launched as the band GEMM's programmatic dependent in the fused step)
    if (R.spec_maxw && ((int)((R.spec_maxw[0] + 9) / 8) != R.spec_sa || (int)((R.spec_maxw[1] + 9) / 8) != R.spec_sb))
        return;  // speculation void (the GEMM stood down too)
    uint32_t* row = sm + threadIdx.x * STR;
    const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t jr = u & 3, i = (u >> 2) % R.M, jq = (u >> 2) / R.M;
    const int64_t j = 4 * jq + jr;
    if (jq * 4 >= R.N || j >= R.N) return;
    const int64_t t = i * R.N + j;
    const size_t plane = (size_t)R.Mp * R.Np;
    const size_t off = rc_off(R, i, j);
    const int NB = R.nwords;
#ifndef APB_RC16_RB
#define APB_RC16_RB 8
#endif
    constexpr int RB = APB_RC16_RB;  // band loads in flight per thread
    uint32_t Wd[NW];
#pragma unroll
    for (int q = 0; q < NW; q++) Wd[q] = 0;
    int32_t run = 0, prev_c = 0;
    bool neg = false;
    // band planes by pointer stepping (one 64-bit add per band, no per-band multiply)
    const uint32_t* pw = R.Tw + off;
    const int32_t* pc = R.Tc + off;
    const uint32_t* pw2 = pw + (size_t)NB * plane;  // SPLIT: planes of the second K split
    const int32_t* pc2 = pc + (size_t)NB * plane;
    constexpr bool v40 = V40;  // Tc is a byte plane: bits 32..39 of the band values
    const int8_t* pb = (const int8_t*)R.Tc + off;
    const int8_t* pb2 = pb + (size_t)NB * plane;
#pragma unroll
    for (int kb = 0; kb < ND; kb += RB) {
        uint32_t w[RB];
        int32_t c[RB];
#pragma unroll
        for (int v = 0; v < RB; v++) {
            const int b = kb + v;
            const bool live = b < NBC && b < NB;
            w[v] = live ? __ldcs(pw) : 0u;
            c[v] = !live ? 0 : v40 ? (int32_t)(int8_t)__ldcs(pb) : __ldcs(pc);
            if (b < NBC) {
                pw += plane;
                if (v40) pb += plane;
                else pc += plane;
            }
        }
        if (SPLIT) {  // raw mode with K split in two: the second split's accumulators, loaded in the
                      // same batch (the sums are the unsplit diagonals, below 2^31 like them)
            uint32_t w2[RB];
            int32_t c2[RB];
#pragma unroll
            for (int v = 0; v < RB; v++) {
                const int b = kb + v;
                const bool live = b < NBC && b < NB;
                w2[v] = live ? __ldcs(pw2) : 0u;
                c2[v] = !live ? 0 : v40 ? (int32_t)(int8_t)__ldcs(pb2) : __ldcs(pc2);
                if (b < NBC) {
                    pw2 += plane;
                    if (v40) pb2 += plane;
                    else pc2 += plane;
                }
            }
#pragma unroll
            for (int v = 0; v < RB; v++) {
                if (v40) {  // low words add with a carry into the high parts
                    const uint32_t t = w[v] + w2[v];
                    c[v] += c2[v] + (t < w[v] ? 1 : 0);
                    w[v] = t;
                } else {
                    w[v] += w2[v];
                    c[v] += c2[v];
                }
            }
        }
        if (R.raw) {
#pragma unroll
            for (int v = 0; v < RB; v++) {
                const int k = kb + v;
                if (k < ND) {
                    // |D| < 2^31: the band value needs 41 bits, the running carry stays below 2^26
                    const int64_t d = v40 ? (int64_t)(((uint64_t)(uint32_t)c[v] << 32) | w[v]) + (int64_t)run
                                          : (int64_t)c[v] * 256 + ((int64_t)run + (int64_t)(int32_t)w[v]);
                    if (k == ND - 1) neg = d < 0;
                    else run = (int32_t)(d >> 16);
                    Wd[k >> 1] |= ((uint32_t)d & 0xFFFFu) << (16 * (k & 1));
                }
            }
        } else {
#pragma unroll
            for (int v = 0; v < RB; v++) {
                const int k = kb + v;
                if (k < ND) {
                    const int32_t d = run + (int32_t)w[v] + prev_c;
                    prev_c = c[v];
                    if (k == ND - 1) neg = d < 0;  // the arithmetic top digit carries the sign
                    else run = d >> 16;
                    Wd[k >> 1] |= ((uint32_t)d & 0xFFFFu) << (16 * (k & 1));
                }
            }
        }
    }
    if (neg) {  // sign-fill above the top digit, then the magnitude
        if (ND & 1) Wd[NW - 1] |= 0xFFFF0000u;
        uint32_t cc = 1;
#pragma unroll
        for (int q = 0; q < NW; q++) {
            const uint32_t v = ~Wd[q] + cc;
            cc = (cc && v == 0) ? 1u : 0u;
            Wd[q] = v;
        }
    }
    // bit length of the magnitude and its words in shared memory (guards at [-1], [NW])
    int top_w = -1;
#pragma unroll
    for (int q = 0; q < NW; q++) {
        row[q + 1] = Wd[q];
        if (Wd[q]) top_w = q;
    }
    row[0] = 0;
    row[NW + 1] = 0;
    BallsOut& O = R.C;
    uint64_t* dst = O.mant + t * (int64_t)O.L;
    Mag rsum = mag_zero();
    if (R.r1b) rsum = mag_add(mag_load(R.r1b[t], R.r1f[t]), mag_load(R.r2b[t], R.r2f[t]));
    if (top_w < 0) {  // exact zero: C stays Ball::zero() (plus the radius products)
        for (int q = 0; q < O.L; q++) dst[q] = 0;
        O.exp[t] = 0;
        O.kind[t] = APB_ZERO;
        mag_store(rsum, &O.rad_man[t], &O.rad_exp[t]);
        return;
    }
    const int64_t B = 32 * (int64_t)top_w + (int64_t)(32 - __clz(row[top_w + 1]));
    // 32 bits of the magnitude starting at bit pos (zeros outside)
    auto bits32 = [&](int64_t pos) -> uint32_t {
        if (pos <= -32 || pos >= 32 * (int64_t)NW) return 0u;
        const int64_t wi = pos >= 0 ? pos >> 5 : -1;
        const int bo = (int)(pos - 32 * wi);
        const uint32_t lo = row[wi + 1], hi = row[wi + 2];
        return bo ? (lo >> bo) | (hi << (32 - bo)) : lo;
    };
    const int64_t exp2 = -R.escale[i] - R.fscale[j];
    int st = 0;
    const int64_t e = checked_add(exp2, B, &st);  // apfloat_from_bigint_scaled exponent
    const int64_t p = R.prec;
    const int64_t cut = B > p ? B - p : 0;  // bits [0, cut) are truncated
    for (int r = 0; r < O.L; r++) {
        const int64_t lo_bit = B - 64 * (int64_t)(r + 1);
        uint64_t v = (uint64_t)bits32(lo_bit) | ((uint64_t)bits32(lo_bit + 32) << 32);
        if (lo_bit < cut) {
            const int64_t k = cut - lo_bit;
            v = k >= 64 ? 0 : (v & ~((1ull << k) - 1));
        }
        dst[O.L - 1 - r] = v;
    }
    O.exp[t] = e;
    O.kind[t] = (uint8_t)(APB_FINITE | (neg ? APB_SIGN : 0));
    // truncation error: Mag upper bound of the discarded bits [0, cut)
    Mag err = mag_zero();
    if (cut > 0) {
        int64_t top = -1;  // highest set bit below the cut
        int64_t q = (cut - 1) >> 5;
        uint32_t m = row[q + 1] & (((cut - 32 * q) >= 32) ? 0xFFFFFFFFu : ((1u << (cut - 32 * q)) - 1u));
        while (true) {
            if (m) {
                top = 32 * q + 31 - __clz(m);
                break;
            }
            if (q == 0) break;
            q--;
            m = row[q + 1];
        }
        if (top >= 0) {
            const int64_t wpos = top - 63;  // 64-bit window with its MSB at `top`
            const uint64_t window = (uint64_t)bits32(wpos) | ((uint64_t)bits32(wpos + 32) << 32);
            bool low = (window & ((1ull << 34) - 1)) != 0;
            if (!low && wpos > 0) {  // any set bit in [0, wpos)
                int64_t qq = (wpos - 1) >> 5;
                uint32_t mm = row[qq + 1] & (((wpos - 32 * qq) >= 32) ? 0xFFFFFFFFu : ((1u << (wpos - 32 * qq)) - 1u));
                while (!mm && qq > 0) {
                    qq--;
                    mm = row[qq + 1];
                }
                low = mm != 0;
            }
            uint64_t bm = window >> 34;
            if (low) bm++;
            err = mag_parts(bm, checked_add(exp2, top + 1, &st));
        }
    }
    if (R.r1b) err = mag_add(err, rsum);
    mag_store(err, &O.rad_man[t], &O.rad_exp[t]);
    if (st) *R.status = st;
}


// ------------------------------------------------ IMAD-limb baseline (K5')
// The same exact block product on CUDA cores, the alternative the north star
// weighs the int8 slices against: scaled integers as sign-magnitude 32-bit limb
// planes, one thread per output entry, Q x Q IMAD.WIDE.U32 limb products per
// term into 2Q signed 64-bit column sums (|sum| < K 2^32 Q), carried into two's
// complement limbs at the end.  Used for measurement (apb_block_int_product_imad)
// and checked against the tensor-core product bit for bit.

// magnitude limbs of mid * 2^scale: A planes [q][r][kk] (rows x w), B planes [q][kk][j] (w x N)
template <int Q>
__global__ void __launch_bounds__(256) limb_pack_kernel(BallsView X, int64_t rows, int64_t cols, int64_t ld,
                                                        int64_t lo, int a_side, const int64_t* top,
                                                        const int64_t* bot, uint32_t* out, uint8_t* sgn,
                                                        int64_t* scale_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= rows * cols) return;
    const int64_t r = t / cols, c = t % cols;  // A: (row, kk); B: (kk, col)
    const int64_t line = a_side ? r : c;
    const int64_t sc = top[line] == INT64_MIN ? 0 : -bot[line];
    if (scale_out && (a_side ? c == 0 : r == 0)) scale_out[line] = sc;
    const int64_t e = a_side ? r * ld + lo + c : (lo + r) * ld + c;
    const uint8_t kd = X.kind[e];
    const bool live = (kd & APB_KIND_MASK) == APB_FINITE;
    const int L = X.L;
    const int64_t sh = live ? X.exp[e] - 64 * (int64_t)L + sc : 0;
    const int64_t lq = (-sh) >> 6;
    const int bo = (int)((-sh) & 63);
    const uint64_t* m = X.mant + e * (int64_t)L;
    const size_t plane = (size_t)rows * cols;
#pragma unroll
    for (int q2 = 0; q2 < (Q + 1) / 2; q2++) {
        const int64_t li = q2 + lq;
        const uint64_t g0 = (live && li >= 0 && li < L) ? m[li] : 0ull;
        const uint64_t g1 = (live && li + 1 >= 0 && li + 1 < L) ? m[li + 1] : 0ull;
        const uint64_t wv = bo ? (g0 >> bo) | (g1 << (64 - bo)) : g0;
        out[(size_t)(2 * q2) * plane + t] = (uint32_t)wv;
        if (2 * q2 + 1 < Q) out[(size_t)(2 * q2 + 1) * plane + t] = (uint32_t)(wv >> 32);
    }
    sgn[t] = live && (kd & APB_SIGN) ? 1 : 0;
}

template <int Q, int TM, int TN>
__global__ void __launch_bounds__(256) imad_gemm_kernel(const uint32_t* __restrict__ Al, const uint8_t* __restrict__ As,
                                                        const uint32_t* __restrict__ Bl, const uint8_t* __restrict__ Bs,
                                                        int64_t M, int64_t N, int64_t w, uint64_t* out, int out_limbs) {
    // 16 x 16 threads, each TM x TN outputs (rows ty + 16 r, cols tx + 16 c); K staged
    // through shared memory KT terms at a time (limb planes [q][kk][row|col])
    constexpr int KT = 8, BM_ = 16 * TM, BN_ = 16 * TN;
    __shared__ uint32_t sa[Q][KT][BM_];
    __shared__ uint32_t sb[Q][KT][BN_];
    __shared__ uint8_t ssa[KT][BM_], ssb[KT][BN_];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.y * BM_, j0 = (int64_t)blockIdx.x * BN_;
    const size_t pa = (size_t)M * w, pb = (size_t)w * N;
    int64_t acc[TM][TN][2 * Q];
#pragma unroll
    for (int r = 0; r < TM; r++)
#pragma unroll
        for (int c = 0; c < TN; c++)
#pragma unroll
            for (int q = 0; q < 2 * Q; q++) acc[r][c][q] = 0;
    for (int64_t k0 = 0; k0 < w; k0 += KT) {
        __syncthreads();
        for (int e = threadIdx.x; e < KT * BM_; e += 256) {  // A: (row, kk), kk fastest (contiguous in k)
            const int kk = e % KT, row = e / KT;
            const int64_t i = i0 + row, k = k0 + kk;
            const bool ok = i < M && k < w;
#pragma unroll
            for (int q = 0; q < Q; q++) sa[q][kk][row] = ok ? __ldg(Al + q * pa + i * w + k) : 0u;
            ssa[kk][row] = ok ? __ldg(As + i * w + k) : 0;
        }
        for (int e = threadIdx.x; e < KT * BN_; e += 256) {  // B: (kk, col), col fastest
            const int col = e % BN_, kk = e / BN_;
            const int64_t j = j0 + col, k = k0 + kk;
            const bool ok = j < N && k < w;
#pragma unroll
            for (int q = 0; q < Q; q++) sb[q][kk][col] = ok ? __ldg(Bl + q * pb + k * N + j) : 0u;
            ssb[kk][col] = ok ? __ldg(Bs + k * N + j) : 0;
        }
        __syncthreads();
#pragma unroll 2
        for (int kk = 0; kk < KT; kk++) {
            uint32_t a[TM][Q], bb[TN][Q];
            int64_t sgn_a[TM], sgn_b[TN];
#pragma unroll
            for (int r = 0; r < TM; r++) {
#pragma unroll
                for (int q = 0; q < Q; q++) a[r][q] = sa[q][kk][ty + 16 * r];
                sgn_a[r] = ssa[kk][ty + 16 * r];
            }
#pragma unroll
            for (int c = 0; c < TN; c++) {
#pragma unroll
                for (int q = 0; q < Q; q++) bb[c][q] = sb[q][kk][tx + 16 * c];
                sgn_b[c] = ssb[kk][tx + 16 * c];
            }
#pragma unroll
            for (int r = 0; r < TM; r++)
#pragma unroll
                for (int c = 0; c < TN; c++) {
                    const int64_t msk = -(sgn_a[r] ^ sgn_b[c]);
#pragma unroll
                    for (int qa = 0; qa < Q; qa++)
#pragma unroll
                        for (int qb = 0; qb < Q; qb++) {
                            const uint64_t p = (uint64_t)a[r][qa] * bb[c][qb];
                            acc[r][c][qa + qb] += (((int64_t)(p & 0xFFFFFFFFull)) ^ msk) - msk;
                            acc[r][c][qa + qb + 1] += (((int64_t)(p >> 32)) ^ msk) - msk;
                        }
                }
        }
    }
    // column sums -> two's complement 32-bit words -> 64-bit limbs (the carry out of
    // the last column still holds magnitude bits: keep emitting it)
#pragma unroll
    for (int r = 0; r < TM; r++)
#pragma unroll
        for (int c = 0; c < TN; c++) {
            const int64_t i = i0 + ty + 16 * r, j = j0 + tx + 16 * c;
            if (i >= M || j >= N) continue;
            uint64_t* dst = out + (size_t)(i * N + j) * out_limbs;
            int64_t carry = 0;
            uint64_t lw = 0;
            int li = 0;
            for (int q = 0; li < out_limbs; q++) {
                const int64_t v = (q < 2 * Q ? acc[r][c][q] : 0) + carry;
                const uint64_t wd = (uint64_t)v & 0xFFFFFFFFull;
                carry = v >> 32;
                if (q & 1) dst[li++] = lw | (wd << 32);
                else lw = wd;
            }
        }
}

// ------------------------------------------------------------ K7 radius
// Mag planes of the four radius operands (src/matmul.cpp:498-509)
APB_DEV Mag mid_upper(const BallsView& a, int64_t e) {
    if ((a.kind[e] & APB_KIND_MASK) != APB_FINITE) return mag_zero();
    return mag_parts((a.mant[e * (int64_t)a.L + a.L - 1] >> 34) + 1, a.exp[e]);
}

// which: 0 |A|, 1 R_A, 2 R_B, 3 |B| + R_B
APB_DEV Mag rad_operand(const BallsView& X, int64_t e, int which) {
    switch (which) {
        case 0: return mid_upper(X, e);
        case 1:
        case 2: return mag_load(X.rad_man[e], X.rad_exp[e]);
        default: return mag_add(mid_upper(X, e), mag_load(X.rad_man[e], X.rad_exp[e]));
    }
}

// per-entry Mag windows (mag_window, src/matmul.cpp:123-128) of the radius
// operands, transposed to [row][l] / [col][l] for the greedy split
__global__ void mag_entry_windows_kernel(BallsView A, BallsView B, int64_t M, int64_t K, int64_t N,
                                         int wa, int wb, longlong2* wA, longlong2* wB) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < M * K) {
        Mag m = rad_operand(A, t, wa);
        wA[t] = m.kind == 1 ? make_longlong2(m.f, m.f - 30) : make_longlong2(INT64_MIN, INT64_MAX);
    } else if (t < M * K + K * N) {
        const int64_t u = t - M * K;
        const int64_t j = u / K, l = u % K;
        Mag m = rad_operand(B, l * N + j, wb);
        wB[u] = m.kind == 1 ? make_longlong2(m.f, m.f - 30) : make_longlong2(INT64_MIN, INT64_MAX);
    }
}


// ------------------------------------------------- fused plan scan (K3 + K7)
// One pass over A (rows) and one over B (columns) collects, per line, three
// bit windows with int64 atomics: the midpoint window (planner, scaling) and
// the Mag windows of the two radius operands on that side (|A|, R_A for rows;
// R_B, |B|+R_B for columns), plus specials and entry precision.
struct LineWins {
    int64_t* top[3];
    int64_t* bot[3];
};

APB_DEV void win_merge(int64_t& top, int64_t& bot, int64_t t, int64_t b) {
    top = t > top ? t : top;
    bot = b < bot ? b : bot;
}

// ---- one-pass plan scan, v2: thread per entry, every field loaded up front,
// block reductions into per-(line, chunk) partials (no atomics, no init pass);
// scan_finish_kernel reduces the partials per line.  Same results as
// fused_rows/cols + fused_finish above (kept for the multi-block path).
struct ScanAcc {
    int64_t t[3], b[3], prec, cnt, special;  // cnt = c1 | c2 << 32
};
constexpr int SCAN_FIELDS = 9;

APB_DEV void sacc_init(ScanAcc& a) {
#pragma unroll
    for (int q = 0; q < 3; q++) {
        a.t[q] = INT64_MIN;
        a.b[q] = INT64_MAX;
    }
    a.prec = 0;
    a.cnt = 0;
    a.special = 0;
}

APB_DEV void sacc_merge(ScanAcc& a, const ScanAcc& o) {
#pragma unroll
    for (int q = 0; q < 3; q++) {
        a.t[q] = o.t[q] > a.t[q] ? o.t[q] : a.t[q];
        a.b[q] = o.b[q] < a.b[q] ? o.b[q] : a.b[q];
    }
    a.prec = o.prec > a.prec ? o.prec : a.prec;
    a.cnt += o.cnt;
    a.special |= o.special;
}

APB_DEV void sacc_shfl(ScanAcc& a, int o) {
    ScanAcc x;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        x.t[q] = __shfl_xor_sync(0xffffffffu, a.t[q], o);
        x.b[q] = __shfl_xor_sync(0xffffffffu, a.b[q], o);
    }
    x.prec = __shfl_xor_sync(0xffffffffu, a.prec, o);
    x.cnt = __shfl_xor_sync(0xffffffffu, a.cnt, o);
    x.special = __shfl_xor_sync(0xffffffffu, a.special, o);
    sacc_merge(a, x);
}

APB_DEV int64_t sacc_get(const ScanAcc& a, int f) {
    switch (f) {
        case 0: return a.t[0];
        case 1: return a.b[0];
        case 2: return a.t[1];
        case 3: return a.b[1];
        case 4: return a.t[2];
        case 5: return a.b[2];
        case 6: return a.prec;
        case 7: return a.cnt;
        default: return a.special;
    }
}

APB_DEV void sacc_set(ScanAcc& a, int f, int64_t v) {
    switch (f) {
        case 0: a.t[0] = v; break;
        case 1: a.b[0] = v; break;
        case 2: a.t[1] = v; break;
        case 3: a.b[1] = v; break;
        case 4: a.t[2] = v; break;
        case 5: a.b[2] = v; break;
        case 6: a.prec = v; break;
        case 7: a.cnt = v; break;
        default: a.special = v;
    }
}

// one entry: midpoint window + entry precision, the two radius-operand Mag
// windows of this side with nonzero counts, specials.  A side: |A|, R_A;
// B side: R_B, |B| + R_B (the operands of src/matmul.cpp:498-509)
APB_DEV void scan_entry(const BallsView& X, int64_t e, bool a_side, ScanAcc& acc, Mag* op1 = nullptr,
                        Mag* op2 = nullptr) {
    // read-only loads (__ldg): they may be hoisted above the plane stores of an
    // earlier entry, so a thread's entries are all in flight together
    const uint8_t kd = __ldg(X.kind + e);
    const int64_t ex = __ldg(X.exp + e);
    const uint32_t rb = __ldg(X.rad_man + e);
    const int64_t rexp = __ldg(X.rad_exp + e);
    const uint64_t* m = X.mant + e * (int64_t)X.L;
    const uint64_t mtop = __ldg(m + X.L - 1);
    const uint64_t m0 = __ldg(m);
    const int k = kd & APB_KIND_MASK;
    acc.special |= ((k != APB_ZERO && k != APB_FINITE) || rb == APB_RAD_INF) ? 1 : 0;
    Mag mu = mag_zero();
    if (k == APB_FINITE) {
        int64_t bw;
        if (m0 != 0 || X.L == 1) {
            bw = 64 * (int64_t)X.L - (int64_t)ctz64(m0);
        } else {
            bw = slot_bitwidth(m, X.L);
        }
        const int64_t t = ex, b = ex - bw;
        win_merge(acc.t[0], acc.b[0], t, b);
        acc.prec = bw > acc.prec ? bw : acc.prec;
        mu = mag_parts((mtop >> 34) + 1, ex);
    }
    const Mag r = (rb != 0 && rb != APB_RAD_INF) ? mag_parts(rb, rexp) : mag_zero();
    const Mag o1 = a_side ? mu : r;
    const Mag o2 = a_side ? r : mag_add(mu, r);
    if (op1) {
        *op1 = o1;
        *op2 = o2;
    }
    if (o1.kind == 1) {
        win_merge(acc.t[1], acc.b[1], o1.f, o1.f - 30);
        acc.cnt += 1;
    }
    if (o2.kind == 1) {
        win_merge(acc.t[2], acc.b[2], o2.f, o2.f - 30);
        acc.cnt += 1ll << 32;
    }
}

// uncentred exact double of a radius operand (the planes the scan writes for the
// speculative radius products; used only when every operand exponent is within
// +-kRadUncentred, so products and sums of <= 2^17 terms stay normal and the
// result equals the centred computation of src/matmul.cpp:404-431 scaled by a
// power of two, which the Mag conversion undoes exactly)
constexpr int64_t kRadUncentred = 480;
APB_DEV double uncentred(const Mag& m) {
    return (m.kind == 1 && m.f <= kRadUncentred + 64 && m.f >= -kRadUncentred - 64) ? ldexp((double)m.b, (int)(m.f - 30))
                                                                                      : 0.0;
}

constexpr int SCAN_A_COLS = 512;  // entries of a row per A block (two per thread)
constexpr int SCAN_B_ROWS = 32;   // rows per B block: 32 columns x 8 warps x 4 rows

// blocks [0, nbA): A rows; [nbA, nbA + nbB): B column tiles.  Partials land in
// pa[f][c][i] (A, cA chunks per row) and pb[f][c][j] (B, cB chunks per column).
#ifdef APB_SCAN_MINB  // occupancy experiments (6 blocks per SM: 16.7 -> 15.7 us at config 3, not adopted)
__global__ void __launch_bounds__(256, APB_SCAN_MINB) scan_v2_kernel(BallsView A, BallsView B, int64_t M, int64_t K, int64_t N,
#else
__global__ void __launch_bounds__(256) scan_v2_kernel(BallsView A, BallsView B, int64_t M, int64_t K, int64_t N,
#endif
                                                      int cA, int cB, int64_t* pa, int64_t* pb, ScanSummary* sum,
                                                      long long* mw1, long long* mw2, double* da1T = nullptr,
                                                      double* da2 = nullptr, double* db1 = nullptr,
                                                      double* db2 = nullptr) {
    __shared__ int64_t red[8][32][SCAN_FIELDS + 1];
    griddep_launch();  // the finish kernel may be scheduled now (it waits for this grid)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the finish kernel accumulates into these
        *sum = ScanSummary{};
        for (int q = 0; q < 4; q++) mw1[q] = mw2[q] = 0;
    }
    const int64_t nbA = M * cA;
    ScanAcc acc;
    sacc_init(acc);
    if ((int64_t)blockIdx.x < nbA) {
        const int64_t i = blockIdx.x / cA;
        const int c = (int)(blockIdx.x % cA);
#pragma unroll
        for (int h = 0; h < SCAN_A_COLS / 256; h++) {
            const int64_t k = (int64_t)c * SCAN_A_COLS + 256 * h + threadIdx.x;
            if (k < K) {
                Mag o1, o2;
                scan_entry(A, i * K + k, true, acc, &o1, &o2);
                if (da1T) {  // |A| transposed ([k][i]) and R_A, uncentred
                    da1T[k * M + i] = uncentred(o1);
                    da2[i * K + k] = uncentred(o2);
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sacc_shfl(acc, o);
        if (lane == 0)
            for (int f = 0; f < SCAN_FIELDS; f++) red[warp][0][f] = sacc_get(acc, f);
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < 8; w++) {
                ScanAcc o;
                for (int f = 0; f < SCAN_FIELDS; f++) sacc_set(o, f, red[w][0][f]);
                sacc_merge(acc, o);
            }
            const int64_t stride = (int64_t)cA * M;
            for (int f = 0; f < SCAN_FIELDS; f++) pa[f * stride + (int64_t)c * M + i] = sacc_get(acc, f);
        }
    } else {
        const int64_t bb = (int64_t)blockIdx.x - nbA;
        const int64_t nct = (N + 31) / 32;
        const int64_t jt = bb % nct;
        const int c = (int)(bb / nct);
        const int64_t j = jt * 32 + lane;
        if (j < N) {
#pragma unroll
            for (int u = 0; u < SCAN_B_ROWS / 8; u++) {
                const int64_t k = (int64_t)c * SCAN_B_ROWS + warp + 8 * u;
                if (k < K) {
                    Mag o1, o2;
                    scan_entry(B, k * N + j, false, acc, &o1, &o2);
                    if (db1) {  // R_B and |B| + R_B, uncentred
                        db1[k * N + j] = uncentred(o1);
                        db2[k * N + j] = uncentred(o2);
                    }
                }
            }
        }
        for (int f = 0; f < SCAN_FIELDS; f++) red[warp][lane][f] = sacc_get(acc, f);
        __syncthreads();
        if (warp == 0 && j < N) {
            for (int w = 1; w < 8; w++) {
                ScanAcc o;
                for (int f = 0; f < SCAN_FIELDS; f++) sacc_set(o, f, red[w][lane][f]);
                sacc_merge(acc, o);
            }
            const int64_t stride = (int64_t)cB * N;
            for (int f = 0; f < SCAN_FIELDS; f++) pb[f * stride + (int64_t)c * N + j] = sacc_get(acc, f);
        }
    }
}

// per line: reduce the chunk partials; rows -> rtop/rbot, centring exponents of
// the two radius operands, maxw_a / special_a / prec_a, radius window widths
// (mw1[0], mw2[0]) and nonzero counts (mw1[2], mw2[2]); columns likewise with
// index 1 / 3.  Threads [0, Mpad) take rows, the rest columns (warp-uniform side).
__global__ void scan_v2_finish_kernel(const int64_t* pa, const int64_t* pb, int64_t M, int64_t N, int cA, int cB,
                                      int64_t* rtop, int64_t* rbot, int64_t* ctop, int64_t* cbot,
                                      int64_t* ecen1, int64_t* ecen2, int64_t* fcen1, int64_t* fcen2,
                                      ScanSummary* sum, long long* mw1, long long* mw2) {
    // warp per line (rows of A first, then columns of B), lanes over the chunk partials;
    // the summary maxima / counts are reduced per block in shared memory first (one set
    // of global atomics per block instead of per line)
    __shared__ long long red[2][8];  // per side: special, far, prec, w0, w1, w2, n1, n2
    griddep_launch();
    if (threadIdx.x < 16) red[threadIdx.x >> 3][threadIdx.x & 7] = 0;
    __syncthreads();
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (wid < M + N) {
        const bool a_side = wid < M;
        const int64_t line = a_side ? wid : wid - M;
        const int64_t n = a_side ? M : N;
        const int nc = a_side ? cA : cB;
        const int64_t* P = a_side ? pa : pb;
        const int64_t stride = (int64_t)nc * n;
        ScanAcc acc;
        sacc_init(acc);
        for (int c = lane; c < nc; c += 32) {
            ScanAcc o;
#pragma unroll
            for (int f = 0; f < SCAN_FIELDS; f++) sacc_set(o, f, P[f * stride + (int64_t)c * n + line]);
            sacc_merge(acc, o);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sacc_shfl(acc, o);
        if (lane == 0) {
            (a_side ? rtop : ctop)[line] = acc.t[0];
            (a_side ? rbot : cbot)[line] = acc.b[0];
            (a_side ? ecen1 : fcen1)[line] = acc.t[1] == INT64_MIN ? 0 : -((acc.t[1] + acc.b[1]) / 2);
            (a_side ? ecen2 : fcen2)[line] = acc.t[2] == INT64_MIN ? 0 : -((acc.t[2] + acc.b[2]) / 2);
            bool far = false;  // operand Mag exponents: f in [b + 30, t] per operand window
            for (int q = 1; q < 3; q++)
                if (acc.t[q] != INT64_MIN && (acc.t[q] > kRadUncentred || acc.b[q] + 30 < -kRadUncentred))
                    far = true;
            long long* r = red[a_side ? 0 : 1];
            if (acc.special) atomicMax(&r[0], 1ll);
            if (far) atomicMax(&r[1], 1ll);
            if (acc.prec) atomicMax(&r[2], (long long)acc.prec);
            if (acc.t[0] != INT64_MIN) atomicMax(&r[3], (long long)(acc.t[0] - acc.b[0]));
            if (acc.t[1] != INT64_MIN) atomicMax(&r[4], (long long)(acc.t[1] - acc.b[1]));
            if (acc.t[2] != INT64_MIN) atomicMax(&r[5], (long long)(acc.t[2] - acc.b[2]));
            atomicAdd((unsigned long long*)&r[6], (unsigned long long)(acc.cnt & 0xffffffffll));
            atomicAdd((unsigned long long*)&r[7], (unsigned long long)(acc.cnt >> 32));
        }
    }
    __syncthreads();
    if (threadIdx.x < 2) {
        const int sd = threadIdx.x;  // 0: A rows, 1: B columns
        const long long* r = red[sd];
        if (r[0]) atomicOr(sd ? &sum->special_b : &sum->special_a, 1);
        if (r[1]) atomicOr(&sum->rad_centred, 1);
        if (r[2]) atomicMax(sd ? &sum->prec_b : &sum->prec_a, r[2]);
        if (r[3]) atomicMax(sd ? &sum->maxw_b : &sum->maxw_a, r[3]);
        if (r[4]) atomicMax(&mw1[sd], r[4]);
        if (r[5]) atomicMax(&mw2[sd], r[5]);
        if (r[6]) atomicAdd((unsigned long long*)&mw1[2 + sd], (unsigned long long)r[6]);
        if (r[7]) atomicAdd((unsigned long long*)&mw2[2 + sd], (unsigned long long)r[7]);
    }
}

// exact double planes of both radius products + nonzero counts, one pass per side
// A side: p1 = |A| (ecen1), p2 = R_A (ecen2);  B side: p1 = R_B (fcen1), p2 = |B|+R_B (fcen2)
__global__ void fused_planes_kernel(BallsView X, int64_t rows, int64_t cols, int a_side, const int64_t* cen1,
                                    const int64_t* cen2, double* p1, double* p2, long long* nz1,
                                    long long* nz2) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double v1 = 0.0, v2 = 0.0;
    if (t < rows * cols) {
        const int64_t line = a_side ? t / cols : t % cols;  // A: row i; B: column j
        Mag m1 = rad_operand(X, t, a_side ? 0 : 2);
        Mag m2 = rad_operand(X, t, a_side ? 1 : 3);
        if (m1.kind == 1) v1 = ldexp((double)m1.b, (int)(m1.f - 30 + cen1[line]));
        if (m2.kind == 1) v2 = ldexp((double)m2.b, (int)(m2.f - 30 + cen2[line]));
        // A side: |A| plane stored transposed ([l][i]) for coalesced column-list products
        if (a_side) p1[(t % cols) * rows + t / cols] = v1;
        else p1[t] = v1;
        p2[t] = v2;
    }
    if (nz1) {
        const unsigned a1 = __ballot_sync(0xffffffffu, v1 != 0.0), a2 = __ballot_sync(0xffffffffu, v2 != 0.0);
        if ((threadIdx.x & 31) == 0) {
            if (a1) atomicAdd((unsigned long long*)nz1, (unsigned long long)__popc(a1));
            if (a2) atomicAdd((unsigned long long*)nz2, (unsigned long long)__popc(a2));
        }
    }
}

// per-row (A side) or per-column (B side) Mag windows over l in [lo,hi)
// -> centring exponent -((top+bot)/2) (src/matmul.cpp:397-411)
__global__ void rad_center_rows_kernel(BallsView A, int64_t M, int64_t K, int64_t lo, int64_t hi,
                                       int which, int64_t* ecen, long long* maxw) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= M) return;
    int64_t top = INT64_MIN, bot = INT64_MAX;
    for (int64_t l = lo + lane; l < hi; l += 32) {
        Mag m = rad_operand(A, i * K + l, which);
        if (m.kind != 1) continue;
        top = m.f > top ? m.f : top;
        bot = (m.f - 30) < bot ? (m.f - 30) : bot;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        int64_t t2 = __shfl_xor_sync(0xffffffffu, top, o);
        int64_t b2 = __shfl_xor_sync(0xffffffffu, bot, o);
        top = t2 > top ? t2 : top;
        bot = b2 < bot ? b2 : bot;
    }
    if (lane == 0) {
        ecen[i] = top == INT64_MIN ? 0 : -((top + bot) / 2);
        if (maxw && top != INT64_MIN) atomicMax(maxw, (long long)(top - bot));
    }
}

__global__ void rad_cols_minmax_kernel(BallsView B, int64_t K, int64_t N, int64_t lo, int64_t hi,
                                       int which, int64_t* ctop, int64_t* cbot) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t k0 = lo + (int64_t)blockIdx.y * COL_CHUNK;
    const int64_t k1 = k0 + COL_CHUNK < hi ? k0 + COL_CHUNK : hi;
    if (j >= N) return;
    int64_t top = INT64_MIN, bot = INT64_MAX;
    for (int64_t l = k0; l < k1; l++) {
        Mag m = rad_operand(B, l * N + j, which);
        if (m.kind != 1) continue;
        top = m.f > top ? m.f : top;
        bot = (m.f - 30) < bot ? (m.f - 30) : bot;
    }
    if (top != INT64_MIN) {
        atomicMax((long long*)&ctop[j], (long long)top);
        atomicMin((long long*)&cbot[j], (long long)bot);
    }
}

__global__ void rad_cols_center_kernel(const int64_t* ctop, const int64_t* cbot, int64_t N,
                                       int64_t* fcen, long long* maxw) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    long long w = 0;
    if (j < N) {
        const int64_t top = ctop[j], bot = cbot[j];
        fcen[j] = top == INT64_MIN ? 0 : -((top + bot) / 2);
        if (top != INT64_MIN) w = (long long)(top - bot);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        long long w2 = __shfl_xor_sync(0xffffffffu, w, o);
        w = w2 > w ? w2 : w;
    }
    if (maxw && (threadIdx.x & 31) == 0 && w) atomicMax(maxw, w);
}

// exact doubles of the centred Mags (mag_ldexp, src/mag.cpp:166-172):
// A side da[i][l] (row-major, width w), B side db[l][j]
__global__ void rad_planes_kernel(BallsView X, int64_t rows, int64_t cols, int64_t lo, int64_t hi,
                                  int which, int a_side, const int64_t* cen, double* out) {
    const int64_t w = hi - lo;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (a_side) {
        if (t >= rows * w) return;
        const int64_t i = t / w, l = t % w;
        Mag m = rad_operand(X, i * cols + lo + l, which);
        out[t] = m.kind == 0 ? 0.0 : ldexp((double)m.b, (int)(m.f - 30 + cen[i]));
    } else {
        if (t >= w * cols) return;
        const int64_t l = t / cols, j = t % cols;
        Mag m = rad_operand(X, (lo + l) * cols + j, which);
        out[t] = m.kind == 0 ? 0.0 : ldexp((double)m.b, (int)(m.f - 30 + cen[j]));
    }
}

// rounded-to-nearest sums in the reference's order, 1024-term chunks, then
// Mag::from_double_upper * (1 + 2^-29) and mag_add_up into r (src/matmul.cpp:423-435).
// 64x64 output tile per 256 threads, 4x4 per thread, sequential in l per entry.
// which radius-product kernel a (speculatively launched) set of candidates
// runs, decided on the device from the scan's nonzero counts mw[2] (A side)
// and mw[3] (B side) with the host's rule (radius_compute): 0 sparse columns
// of Q, 1 sparse rows of P, 2 dense.  Bit-identical results either way.
__host__ __device__ inline int rad_variant(const long long* mw, int64_t M, int64_t K, int64_t N, int a_trans) {
    const double dens_a = M * K ? (double)mw[2] / (double)(M * K) : 1.0;
    const double dens_b = K * N ? (double)mw[3] / (double)(K * N) : 1.0;
    if (a_trans && dens_b <= 0.25 && dens_b <= dens_a) return 0;
    if (!a_trans && dens_a <= 0.25) return 1;
    return 2;
}

constexpr int RT = 32, RK = 32, RTHREADS = 64;
#ifndef APB_RADG_UNROLL
#define APB_RADG_UNROLL 4
#endif
constexpr int RADG_UNROLL = APB_RADG_UNROLL;  // k steps of a full tile unrolled together
static_assert(RT == RK, "the transposed A-tile fetch of rad_gemm_body maps k and row indices through RT");
// PT x PT outputs per thread: PT = 4 (64 threads per 32 x 32 tile) for large
// products, PT = 2 (256 threads) when the grid is too small to fill the SMs with
// the 64-thread tiles (c2: 128 tiles, ~2 warps per SM, FP64 latency-bound)
template <int PT>
APB_DEV void rad_gemm_body(const double* __restrict__ da, const double* __restrict__ db, int64_t M, int64_t N,
                           int64_t w, const int64_t* ecen, const int64_t* fcen, uint32_t* rb, int64_t* rf,
                           int accumulate, int a_trans, const long long* sel, int64_t bx, int64_t by,
                           const int* cflag = nullptr) {
    if (sel && rad_variant(sel, M, w, N, a_trans) != 2) return;
    const bool cen = !cflag || *cflag;  // uncentred planes (scan-written) unless flagged
    // 32 x 32 outputs per 64 threads (4 x 4 each), K tiles of 32 staged in shared
    // memory with the next tile prefetched into registers; per-entry sequential RN
    // sums (__dmul_rn / __dadd_rn, no contraction) folded into the Mag bound at
    // every 1024-term chunk end (src/matmul.cpp:404-431); the folded Mags wait in
    // shared memory (they are touched once per chunk)
    // rows 16-byte aligned: 128-bit operand loads.  The once-per-tile transposed
    // store sA[q % RT][q / RT] of a row-major A plane puts lanes r, r+8, r+16, r+24
    // on one bank pair (4 wavefronts for 32 doubles instead of 2); with even row
    // strides and pair-preserving swizzles every lane's double has the same slot
    // parity, so the 2-wavefront minimum needs odd strides, which would break the
    // double2 loads of the inner loop (the hot part) -- accepted.
    __shared__ __align__(16) double sA[RK][RT + 2];
    __shared__ __align__(16) double sB[RK][RT];
    // column permutation of the B tile for PT = 4: a thread's four columns 4 tx .. 4 tx + 3 are read as
    // two 16-byte loads; stored in place the 8 threads of a row would read 16-byte pieces 32 bytes apart
    // (tx and tx + 4 on the same banks: ncu counted 2 extra wavefronts per shared load at N = 1024), so
    // the pair (h / 2) of thread tx lives at 16-byte slot (h / 2) * 8 + tx: 8 threads x 16 B contiguous
    auto bcol = [](int c) -> int { return PT == 4 ? ((((c & 3) >> 1) * 8 + (c >> 2)) << 1) | (c & 1) : c; };
    constexpr int NT = (RT / PT) * (RT / PT);  // threads per tile
    __shared__ uint32_t eb[PT * PT][NT];
    __shared__ int64_t ef[PT * PT][NT];
    constexpr int PER = RK * RT / NT;  // tile elements per thread per operand
    const int tx = threadIdx.x % (RT / PT), ty = threadIdx.x / (RT / PT);
    const int64_t i0 = by * RT, j0 = bx * RT;
    double s[PT][PT];
#pragma unroll
    for (int r = 0; r < PT; r++)
#pragma unroll
        for (int c = 0; c < PT; c++) {
            s[r][c] = 0.0;
            eb[PT * r + c][threadIdx.x] = 0;
            ef[PT * r + c][threadIdx.x] = 0;
        }
    const Mag infl = mag_parts((1ull << 29) + 1, 1);
    double pa[PER], pb[PER];
    const bool rows_in = i0 + RT <= M && j0 + RT <= N;
    // A tiles of a row-major plane (a_trans = 0, M x w) are read with consecutive
    // threads along k (coalesced rows) and stored transposed into sA[k][i]
    auto fetch = [&](int64_t l0) {
        if (rows_in && l0 + RK <= w) {  // interior tile: strided pointers, no bounds tests
            // element u: kk = tid / 32 + (NT / 32) u, rr = tid % 32
            const int kk0 = threadIdx.x / RT, rr = threadIdx.x % RT;
            const double* pB = db + (l0 + kk0) * N + j0 + rr;
            const int64_t sb = (int64_t)(NT / RT) * N;
            if (a_trans) {
                const double* pA = da + (l0 + kk0) * M + i0 + rr;
                const int64_t sa = (int64_t)(NT / RT) * M;
#pragma unroll
                for (int u = 0; u < PER; u++) pa[u] = __ldg(pA + u * sa);
            } else {  // element u: row i0 + tid / 32 + (NT / 32) u, k = l0 + tid % 32
                const double* pA = da + (i0 + kk0) * w + l0 + rr;
                const int64_t sa = (int64_t)(NT / RT) * w;
#pragma unroll
                for (int u = 0; u < PER; u++) pa[u] = __ldg(pA + u * sa);
            }
#pragma unroll
            for (int u = 0; u < PER; u++) pb[u] = __ldg(pB + u * sb);
            return;
        }
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int q = threadIdx.x + NT * u;
            const int kk = q / RT, rr = q % RT;
            const int64_t gi = i0 + rr, gl = l0 + kk, gj = j0 + rr;
            if (a_trans)
                pa[u] = (gi < M && gl < w) ? da[gl * M + gi] : 0.0;
            else  // transposed roles: row i0 + kk, k l0 + rr
                pa[u] = (i0 + kk < M && l0 + rr < w) ? da[(i0 + kk) * w + l0 + rr] : 0.0;
            pb[u] = (gj < N && gl < w) ? db[gl * N + gj] : 0.0;
        }
    };
    fetch(0);
    for (int64_t l0 = 0; l0 < w; l0 += RK) {
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; u++) {
            const int q = threadIdx.x + NT * u;
            if (a_trans)
                sA[q / RT][q % RT] = pa[u];
            else
                sA[q % RT][q / RT] = pa[u];
            sB[q / RT][bcol(q % RT)] = pb[u];
        }
        __syncthreads();
        if (l0 + RK < w) fetch(l0 + RK);
        const int kmax = (w - l0) < RK ? (int)(w - l0) : RK;
        auto kstep = [&](int kk) {
            double a[PT], b[PT];
#pragma unroll
            for (int h = 0; h < PT; h += 2) {
                const double2 av = *reinterpret_cast<const double2*>(&sA[kk][ty * PT + h]);
                const double2 bv = *reinterpret_cast<const double2*>(&sB[kk][bcol(tx * PT + h)]);
                a[h] = av.x;
                a[h + 1] = av.y;
                b[h] = bv.x;
                b[h + 1] = bv.y;
            }
#pragma unroll
            for (int r = 0; r < PT; r++)
#pragma unroll
                for (int c = 0; c < PT; c++) s[r][c] = __dadd_rn(s[r][c], __dmul_rn(a[r], b[c]));
        };
        if (kmax == RK) {  // full tile: unrolled so the shared loads of later steps are issued early
#pragma unroll RADG_UNROLL
            for (int kk = 0; kk < RK; kk++) kstep(kk);
        } else {
            for (int kk = 0; kk < kmax; kk++) kstep(kk);
        }
        const int64_t l = l0 + kmax;  // RK divides 1024: chunk ends fall on tile ends
        if ((l & 1023) == 0 || l == w) {
#pragma unroll
            for (int r = 0; r < PT; r++)
#pragma unroll
                for (int c = 0; c < PT; c++) {
                    const int64_t gi = i0 + ty * PT + r, gj = j0 + tx * PT + c;
                    if (s[r][c] != 0.0 && gi < M && gj < N) {
                        const Mag e = mag_add(mag_load(eb[PT * r + c][threadIdx.x], ef[PT * r + c][threadIdx.x]),
                                              mag_mul(mag_from_double(s[r][c], cen ? -ecen[gi] - fcen[gj] : 0), infl));
                        mag_store(e, &eb[PT * r + c][threadIdx.x], &ef[PT * r + c][threadIdx.x]);
                    }
                    s[r][c] = 0.0;
                }
        }
    }
#pragma unroll
    for (int r = 0; r < PT; r++)
#pragma unroll
        for (int c = 0; c < PT; c++) {
            const int64_t gi = i0 + ty * PT + r, gj = j0 + tx * PT + c;
            if (gi >= M || gj >= N) continue;
            const int64_t o = gi * N + gj;
            Mag m = mag_load(eb[PT * r + c][threadIdx.x], ef[PT * r + c][threadIdx.x]);
            if (accumulate) {
                if (m.kind == 0) continue;
                m = mag_add(mag_load(rb[o], rf[o]), m);
            }
            mag_store(m, &rb[o], &rf[o]);
        }
}

__global__ void __launch_bounds__(64) rad_gemm_kernel(const double* __restrict__ da,
                                                       const double* __restrict__ db, int64_t M,
                                                       int64_t N, int64_t w, const int64_t* ecen,
                                                       const int64_t* fcen, uint32_t* rb, int64_t* rf,
                                                       int accumulate, int a_trans, const long long* sel = nullptr) {
    rad_gemm_body<4>(da, db, M, N, w, ecen, fcen, rb, rf, accumulate, a_trans, sel, blockIdx.x, blockIdx.y);
}


// ---- sparse radius products (bit-exact: skipping exact zero terms leaves every
// RN partial sum unchanged since s + (+0.0) == s for s >= 0)
// ordered nonzero lists of a plane: columns of db (w x N) / rows of da (M x w)
__global__ void col_lists_kernel(const double* __restrict__ db, int64_t w, int64_t N, int* cnt, int* idx,
                                 double* val) {
    const int lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= N) return;
    int base = 0;
    for (int64_t l0 = 0; l0 < w; l0 += 32) {
        const int64_t l = l0 + lane;
        const double v = l < w ? db[l * N + j] : 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, v != 0.0);
        if (v != 0.0) {  // list entry p of column j lives at [p][j] (coalesced reads later)
            const int pos = base + __popc(m & ((1u << lane) - 1u));
            idx[(int64_t)pos * N + j] = (int)l;
            val[(int64_t)pos * N + j] = v;
        }
        base += __popc(m);
    }
    if (lane == 0) cnt[j] = base;
}

__global__ void row_lists_kernel(const double* __restrict__ da, int64_t M, int64_t w, int* cnt, int* idx,
                                 double* val, int a_trans) {
    const int lane = threadIdx.x & 31;
    const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (i >= M) return;
    int base = 0;
    for (int64_t l0 = 0; l0 < w; l0 += 32) {
        const int64_t l = l0 + lane;
        const double v = l < w ? (a_trans ? da[l * M + i] : da[i * w + l]) : 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, v != 0.0);
        if (v != 0.0) {
            const int pos = base + __popc(m & ((1u << lane) - 1u));
            idx[i * w + pos] = (int)l;
            val[i * w + pos] = v;
        }
        base += __popc(m);
    }
    if (lane == 0) cnt[i] = base;
}

// mag_mul(mag_from_double(s, x), (1 + 2^-29)) for s > 0: Mag::from_double_upper
// (src/mag.cpp:79-87: 53-bit mantissa -> top 30 bits rounded up) and mag_mul_up
// (src/mag.cpp:132-145) on the double's bit fields; normal doubles and |x| < 2^40 take
// the integer path, everything else the general routines (same results)
APB_DEV Mag rad_fold_mag(double s, int64_t x) {
    const uint64_t bits = (uint64_t)__double_as_longlong(s);
    const int E = (int)(bits >> 52) & 0x7ff;
    if (E == 0 || E == 0x7ff || (bits >> 63) || x > ((int64_t)1 << 40) || x < -((int64_t)1 << 40))
        return mag_mul(mag_from_double(s, x), mag_parts((1ull << 29) + 1, 1));
    const uint64_t m53 = (bits & ((1ull << 52) - 1)) | (1ull << 52);
    uint64_t b = m53 >> 23;
    if (m53 & ((1ull << 23) - 1)) b++;
    int64_t f = x + (int64_t)(E - 1022);
    if (b == kMagOne) {
        b >>= 1;
        f++;
    }
    uint64_t q = (b * ((1ull << 29) + 1) + (kMagOne - 1)) >> 30;
    f += 1;
    if (q < (kMagOne >> 1)) {
        q <<= 1;
        f--;
    }
    return mag_parts(q, f);
}

APB_DEV void rad_fold(Mag& ent, double& s, int64_t e_i, int64_t f_j) {
    if (s != 0.0) ent = mag_add(ent, rad_fold_mag(s, -e_i - f_j));
    s = 0.0;
}

// out(i,j) over the nonzero list of column j of db; warp per (32 rows i, column j):
// list entries are warp-uniform (broadcast), the |A| plane is read transposed
// (daT[l][i], coalesced across the warp)
__global__ void __launch_bounds__(256) rad_spcol_kernel(const double* __restrict__ daT, int64_t M, int64_t N,
                                                        int64_t w, const int* cnt, const int* idx,
                                                        const double* val, const int64_t* ecen,
                                                        const int64_t* fcen, uint32_t* rb, int64_t* rf) {
    const int64_t i = (int64_t)blockIdx.x * 32 + (threadIdx.x & 31);
    const int64_t j = (int64_t)blockIdx.y * 8 + (threadIdx.x >> 5);
    if (j >= N) return;
    double s = 0.0;
    Mag ent = mag_zero();
    int64_t chunk_end = 1024;
    const int n = cnt[j];
    const int64_t ii = i < M ? i : 0;
    for (int p = 0; p < n; p++) {
        const int l = idx[(int64_t)p * N + j];
        const double v = val[(int64_t)p * N + j];
        if (l >= chunk_end) {
            rad_fold(ent, s, ecen[ii], fcen[j]);
            chunk_end = ((int64_t)l / 1024 + 1) * 1024;
        }
        s = __dadd_rn(s, __dmul_rn(daT[(int64_t)l * M + ii], v));
    }
    if (i >= M) return;
    rad_fold(ent, s, ecen[i], fcen[j]);
    mag_store(ent, &rb[i * N + j], &rf[i * N + j]);
}

// out(i,j) over the nonzero list of row i of da; thread per (i, j)
__global__ void __launch_bounds__(256) rad_sprow_kernel(const double* __restrict__ db, int64_t M, int64_t N,
                                                        int64_t w, const int* cnt, const int* idx,
                                                        const double* val, const int64_t* ecen,
                                                        const int64_t* fcen, uint32_t* rb, int64_t* rf) {
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    const int64_t i = blockIdx.y;
    if (j >= N) return;
    double s = 0.0;
    Mag ent = mag_zero();
    int64_t chunk_end = 1024;
    const int n = cnt[i];
    for (int p = 0; p < n; p++) {
        const int l = idx[i * w + p];
        if (l >= chunk_end) {
            rad_fold(ent, s, ecen[i], fcen[j]);
            chunk_end = ((int64_t)l / 1024 + 1) * 1024;
        }
        s = __dadd_rn(s, __dmul_rn(val[i * w + p], db[(int64_t)l * N + j]));
    }
    rad_fold(ent, s, ecen[i], fcen[j]);
    mag_store(ent, &rb[i * N + j], &rf[i * N + j]);
}

// ---- fused list + product, v2: one CTA per column j (spcol) / row i (sprow)
// compacts that line's nonzeros of a 1024-term chunk into shared memory in
// l order (block ballot prefix), then every thread runs its own RN sum over
// the list with the operand loads issued 8 at a time.  Same term order and
// chunk folds as rad_spcol/rad_sprow (bit-identical results).
constexpr int RCH = 1024;

template <int R, int T>
struct RadSmem {
    int sl[RCH];
    double sv[RCH];
    int cnt[65];
    double gbuf[8 * R][T];
};

// ordered compaction of v[u] (term l = c0 + T u + tid, T threads, U = RCH / T) into
// (sl, sv); returns the count.  cnt holds the 32 (u, warp) counts in l order.
template <int T>
APB_DEV int block_compact_t(const double (&v)[RCH / T], int64_t c0, int* sl, double* sv, int* cnt) {
    constexpr int U = RCH / T, NWP = T / 32;
    static_assert(U * NWP == 32, "32 (u, warp) groups");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned bal[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        bal[u] = __ballot_sync(0xffffffffu, v[u] != 0.0);
        if (lane == 0) cnt[u * NWP + warp] = __popc(bal[u]);
    }
    __syncthreads();
    if (warp == 0) {
        const int c = cnt[lane];
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        cnt[32 + lane] = x - c;
        if (lane == 31) cnt[64] = x;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < U; u++) {
        if (v[u] != 0.0) {
            const int pos = cnt[32 + u * NWP + warp] + __popc(bal[u] & ((1u << lane) - 1u));
            sl[pos] = (int)(c0 + T * u + tid);
            sv[pos] = v[u];
        }
    }
    __syncthreads();
    return cnt[64];
}

APB_DEV int block_compact(const double (&v)[4], int64_t c0, int* sl, double* sv, int* cnt) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned bal[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
        bal[u] = __ballot_sync(0xffffffffu, v[u] != 0.0);
        if (lane == 0) cnt[u * 8 + warp] = __popc(bal[u]);
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the 32 (u, warp) counts in l order
        const int c = cnt[lane];
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        cnt[32 + lane] = x - c;
        if (lane == 31) cnt[64] = x;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; u++) {
        if (v[u] != 0.0) {
            const int pos = cnt[32 + u * 8 + warp] + __popc(bal[u] & ((1u << lane) - 1u));
            sl[pos] = (int)(c0 + 256 * u + tid);
            sv[pos] = v[u];
        }
    }
    __syncthreads();
    return cnt[64];
}

// |A| R_B with R_B sparse: CTA per column j of db (w x N); |A| plane transposed daT[l][i]
__global__ void __launch_bounds__(256) rad_spcol_v2_kernel(const double* __restrict__ daT, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf) {
    __shared__ int sl[RCH];
    __shared__ double sv[RCH];
    __shared__ int cnt[65];
    const int64_t j = blockIdx.x;
    const int64_t nch = (w + RCH - 1) / RCH;
    const int64_t fj = fcen[j];
    int n = 0;
    for (int64_t pass = 0; pass * 256 < M; pass++) {
        const int64_t i = pass * 256 + threadIdx.x;
        const int64_t ii = i < M ? i : 0;
        double s = 0.0;
        Mag ent = mag_zero();
        for (int64_t c0 = 0; c0 < w; c0 += RCH) {
            if (nch > 1 || pass == 0) {
                if (nch > 1) __syncthreads();  // previous chunk's list fully consumed
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int64_t l = c0 + 256 * u + threadIdx.x;
                    v[u] = l < w ? db[l * N + j] : 0.0;
                }
                n = block_compact(v, c0, sl, sv, cnt);
            }
            for (int p0 = 0; p0 < n; p0 += 8) {
                double a[8];
#pragma unroll
                for (int u = 0; u < 8; u++) a[u] = p0 + u < n ? daT[(int64_t)sl[p0 + u] * M + ii] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; u++)
                    if (p0 + u < n) s = __dadd_rn(s, __dmul_rn(a[u], sv[p0 + u]));
            }
            rad_fold(ent, s, ecen[ii], fj);
        }
        if (i < M) mag_store(ent, &rb[i * N + j], &rf[i * N + j]);
    }
}

// R_A (|B| + R_B) with R_A sparse: CTA per row i of da (M x w, row-major)
__global__ void __launch_bounds__(256) rad_sprow_v2_kernel(const double* __restrict__ da, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf) {
    __shared__ int sl[RCH];
    __shared__ double sv[RCH];
    __shared__ int cnt[65];
    const int64_t i = blockIdx.x;
    const int64_t nch = (w + RCH - 1) / RCH;
    const int64_t ei = ecen[i];
    int n = 0;
    for (int64_t pass = 0; pass * 256 < N; pass++) {
        const int64_t j = pass * 256 + threadIdx.x;
        const int64_t jj = j < N ? j : 0;
        double s = 0.0;
        Mag ent = mag_zero();
        for (int64_t c0 = 0; c0 < w; c0 += RCH) {
            if (nch > 1 || pass == 0) {
                if (nch > 1) __syncthreads();
                double v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    const int64_t l = c0 + 256 * u + threadIdx.x;
                    v[u] = l < w ? da[i * w + l] : 0.0;
                }
                n = block_compact(v, c0, sl, sv, cnt);
            }
            for (int p0 = 0; p0 < n; p0 += 8) {
                double b[8];
#pragma unroll
                for (int u = 0; u < 8; u++) b[u] = p0 + u < n ? db[(int64_t)sl[p0 + u] * N + jj] : 0.0;
#pragma unroll
                for (int u = 0; u < 8; u++)
                    if (p0 + u < n) s = __dadd_rn(s, __dmul_rn(sv[p0 + u], b[u]));
            }
            rad_fold(ent, s, ei, fcen[jj]);
        }
        if (j < N) mag_store(ent, &rb[i * N + j], &rf[i * N + j]);
    }
}

APB_DEV void cp_async8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(sdst)),
                 "l"(gsrc)
                 : "memory");
}
APB_DEV void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// ---- v3: as v2, with R lines per thread (independent RN sums interleaved for
// ILP, one list read serving R loads); the 8R gathered operands of a batch are
// fetched with cp.async into a per-thread shared-memory column so they are all
// in flight together (the compiler otherwise interleaves each load with its use)
template <int R, int T>
APB_DEV void rad_spcol_v3_body(RadSmem<R, T>& sm, int64_t blk, const double* __restrict__ daT, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf,
                                                           const long long* sel = nullptr, const int* cflag = nullptr) {
    if (sel && rad_variant(sel, M, w, N, 1) != 0) return;
    int* sl = sm.sl;
    double* sv = sm.sv;
    int* cnt = sm.cnt;
    auto& gbuf = sm.gbuf;
    const int64_t j = blk;
    const int64_t nch = (w + RCH - 1) / RCH;
    const bool cen = !cflag || *cflag;  // uncentred planes (scan-written) unless flagged
    const int64_t fj = cen ? fcen[j] : 0;
    int n = 0;
    for (int64_t pass = 0; pass * T * R < M; pass++) {
        int64_t ii[R];
        double s[R];
        Mag ent[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t i = pass * T * R + T * r + threadIdx.x;
            ii[r] = i < M ? i : 0;
            s[r] = 0.0;
            ent[r] = mag_zero();
        }
        for (int64_t c0 = 0; c0 < w; c0 += RCH) {
            if (nch > 1 || pass == 0) {
                if (nch > 1) __syncthreads();
                double v[RCH / T];
#pragma unroll
                for (int u = 0; u < RCH / T; u++) {
                    const int64_t l = c0 + T * u + threadIdx.x;
                    v[u] = l < w ? db[l * N + j] : 0.0;
                }
                n = block_compact_t<T>(v, c0, sl, sv, cnt);
            }
            int p0 = 0;
            for (; p0 + 8 <= n; p0 += 8) {
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double* row = daT + (int64_t)sl[p0 + u] * M;
#pragma unroll
                    for (int r = 0; r < R; r++) cp_async8(&gbuf[u * R + r][threadIdx.x], row + ii[r]);
                }
                cp_async_wait_all();
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double bv = sv[p0 + u];
#pragma unroll
                    for (int r = 0; r < R; r++) s[r] = __dadd_rn(s[r], __dmul_rn(gbuf[u * R + r][threadIdx.x], bv));
                }
            }
            for (; p0 < n; p0++) {
                const double* row = daT + (int64_t)sl[p0] * M;
                const double bv = sv[p0];
#pragma unroll
                for (int r = 0; r < R; r++) s[r] = __dadd_rn(s[r], __dmul_rn(row[ii[r]], bv));
            }
#pragma unroll
            for (int r = 0; r < R; r++) rad_fold(ent[r], s[r], cen ? ecen[ii[r]] : 0, fj);
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t i = pass * T * R + T * r + threadIdx.x;
            if (i < M) mag_store(ent[r], &rb[i * N + j], &rf[i * N + j]);
        }
    }
}

template <int R, int T = 256>
__global__ void __launch_bounds__(T) rad_spcol_v3_kernel(const double* __restrict__ daT, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf,
                                                           const long long* sel = nullptr) {
    __shared__ RadSmem<R, T> sm;
    rad_spcol_v3_body<R, T>(sm, blockIdx.x, daT, db, M, N, w, ecen, fcen, rb, rf, sel);
}

template <int R, int T>
APB_DEV void rad_sprow_v3_body(RadSmem<R, T>& sm, int64_t blk, const double* __restrict__ da, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf,
                                                           const long long* sel = nullptr, const int* cflag = nullptr) {
    if (sel && rad_variant(sel, M, w, N, 0) != 1) return;
    int* sl = sm.sl;
    double* sv = sm.sv;
    int* cnt = sm.cnt;
    auto& gbuf = sm.gbuf;
    const int64_t i = blk;
    const int64_t nch = (w + RCH - 1) / RCH;
    const bool cen = !cflag || *cflag;
    const int64_t ei = cen ? ecen[i] : 0;
    int n = 0;
    for (int64_t pass = 0; pass * T * R < N; pass++) {
        int64_t jj[R];
        double s[R];
        Mag ent[R];
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t j = pass * T * R + T * r + threadIdx.x;
            jj[r] = j < N ? j : 0;
            s[r] = 0.0;
            ent[r] = mag_zero();
        }
        for (int64_t c0 = 0; c0 < w; c0 += RCH) {
            if (nch > 1 || pass == 0) {
                if (nch > 1) __syncthreads();
                double v[RCH / T];
#pragma unroll
                for (int u = 0; u < RCH / T; u++) {
                    const int64_t l = c0 + T * u + threadIdx.x;
                    v[u] = l < w ? da[i * w + l] : 0.0;
                }
                n = block_compact_t<T>(v, c0, sl, sv, cnt);
            }
            int p0 = 0;
            for (; p0 + 8 <= n; p0 += 8) {
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double* row = db + (int64_t)sl[p0 + u] * N;
#pragma unroll
                    for (int r = 0; r < R; r++) cp_async8(&gbuf[u * R + r][threadIdx.x], row + jj[r]);
                }
                cp_async_wait_all();
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const double av = sv[p0 + u];
#pragma unroll
                    for (int r = 0; r < R; r++) s[r] = __dadd_rn(s[r], __dmul_rn(av, gbuf[u * R + r][threadIdx.x]));
                }
            }
            for (; p0 < n; p0++) {
                const double* row = db + (int64_t)sl[p0] * N;
                const double av = sv[p0];
#pragma unroll
                for (int r = 0; r < R; r++) s[r] = __dadd_rn(s[r], __dmul_rn(av, row[jj[r]]));
            }
#pragma unroll
            for (int r = 0; r < R; r++) rad_fold(ent[r], s[r], ei, cen ? fcen[jj[r]] : 0);
        }
#pragma unroll
        for (int r = 0; r < R; r++) {
            const int64_t j = pass * T * R + T * r + threadIdx.x;
            if (j < N) mag_store(ent[r], &rb[i * N + j], &rf[i * N + j]);
        }
    }
}

template <int R, int T = 256>
__global__ void __launch_bounds__(T) rad_sprow_v3_kernel(const double* __restrict__ da, const double* __restrict__ db,
                                                           int64_t M, int64_t N, int64_t w, const int64_t* ecen,
                                                           const int64_t* fcen, uint32_t* rb, int64_t* rf,
                                                           const long long* sel = nullptr) {
    __shared__ RadSmem<R, T> sm;
    rad_sprow_v3_body<R, T>(sm, blockIdx.x, da, db, M, N, w, ecen, fcen, rb, rf, sel);
}

// both radius products of a speculative single block in one launch each
// (src/matmul.cpp:498-513): R1 = |A| R_B (plane 1, |A| transposed) and
// R2 = R_A (|B| + R_B) (plane 2); the device picks sparse / dense (rad_variant)
struct RadPair {
    int64_t M, K, N;
    double *da1, *db1, *da2, *db2;
    const int64_t *ec1, *fc1, *ec2, *fc2;
    uint32_t *r1b, *r2b;
    int64_t *r1f, *r2f;
    const long long *mw1, *mw2;
    const int* cflag;  // nullable: 0 = the scan's uncentred planes are exact (no planes pass)
};

// blocks [0, N): column lists of R_B (product 1); [N, N + M): row lists of R_A (product 2)
template <int R, int T>
__global__ void __launch_bounds__(T) rad_sparse2_kernel(RadPair P) {
    __shared__ RadSmem<R, T> sm;
    if ((int64_t)blockIdx.x < P.N)
        rad_spcol_v3_body<R, T>(sm, blockIdx.x, P.da1, P.db1, P.M, P.N, P.K, P.ec1, P.fc1, P.r1b, P.r1f, P.mw1,
                                P.cflag);
    else
        rad_sprow_v3_body<R, T>(sm, (int64_t)blockIdx.x - P.N, P.da2, P.db2, P.M, P.N, P.K, P.ec2, P.fc2, P.r2b,
                                P.r2f, P.mw2, P.cflag);
}

// ---- tiled sparse products (the speculative step's default).  rad_sparse2 gathers
// every term's dense operand from L2 (26 terms x 8 B per output at config 3, ~109 MB of L2
// reads for both products); here the sparse lines' (index, value) lists are compacted
// once (rad_lists_kernel, warp per line, l order) and a CTA keeps a strip of TI dense
// lines (TI x 1024 doubles per chunk) in shared memory, so a list entry read once
// serves TI outputs: thread = sparse line, TI interleaved RN sums in the reference's
// term order, chunk folds at the 1024-term boundaries (src/matmul.cpp:404-431).
// Zero terms are skipped (s + a 0 = s for the nonnegative finite planes): same bits as
// rad_sparse2 / rad_gemm2.
struct RadLists {
    int *cnt1, *idx1;  // product 1: column lists of db1 (K x N): cnt1[sub-chunk][N] cumulative, idx1[N][K]
    double* val1;
    int *cnt2, *idx2;  // product 2: row lists of da2 (M x K): cnt2[sub-chunk][M], idx2[M][K]
    double* val2;
};
constexpr int RSUB = 256;     // list sub-chunk = dense strip depth in shared memory (RCH = 4 RSUB)
constexpr int RQ_DL = 16;     // dense lines per strip (two per lane): 256 x 16 doubles = 32 KB
constexpr int RQ_WARPS = 8;   // warps per CTA: 2 per SM sub-partition at 88 registers beside a raw band-GEMM CTA
constexpr int RQ_T = 32 * RQ_WARPS;
constexpr int RQ_QW = 4;      // line quads per warp and item
constexpr int RQ_LINES = RQ_WARPS * 4 * RQ_QW;  // sparse lines per item: warps x RQ_QW quads x 4 lines
constexpr int RQ_SMEM = RSUB * RQ_DL * (int)sizeof(double);

__global__ void __launch_bounds__(256) rad_lists_kernel(RadPair P, RadLists L) {
    const int64_t wl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wl >= P.N + P.M) return;
    const bool first = wl < P.N;
    if (first ? rad_variant(P.mw1, P.M, P.K, P.N, 1) != 0 : rad_variant(P.mw2, P.M, P.K, P.N, 0) != 1) return;
    const int64_t line = first ? wl : wl - P.N;
    const int64_t LN = first ? P.N : P.M;
    const double* src = first ? P.db1 + line : P.da2 + line * P.K;
    const int64_t stride = first ? P.N : 1;
    int* cnt = first ? L.cnt1 : L.cnt2;
    int* idx = first ? L.idx1 : L.idx2;
    double* val = first ? L.val1 : L.val2;
    int pos = 0;
    for (int64_t c0 = 0; c0 < P.K; c0 += RSUB) {
        const int64_t c1 = c0 + RSUB < P.K ? c0 + RSUB : P.K;
        double v[RSUB / 32];
#pragma unroll
        for (int u = 0; u < RSUB / 32; u++) {
            const int64_t l = c0 + 32 * u + lane;
            v[u] = l < c1 ? src[l * stride] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RSUB / 32; u++) {
            const unsigned bal = __ballot_sync(0xffffffffu, v[u] != 0.0);
            if (v[u] != 0.0) {
                const int64_t q = pos + __popc(bal & ((1u << lane) - 1u));
                idx[line * P.K + q] = (int)(c0 + 32 * u + lane);
                val[line * P.K + q] = v[u];
            }
            pos += __popc(bal);
        }
        if (lane == 0) cnt[(c0 / RSUB) * LN + line] = pos;
    }
}

// Work item = (strip of 16 dense lines, group of 128 sparse lines); 128-thread CTAs walk
// the items round-robin.  The strip's 256-deep sub-chunk sits in shared memory as [l][16]
// (32 KB: with 128 threads and <= 128 registers a CTA fits beside a raw-epilogue band-GEMM
// CTA, where the speculative step runs it, launched as the GEMM's programmatic dependent).
// A warp takes four sparse lines at a time: lane = (line g = lane / 8, dense lines 2r, 2r+1
// with r = lane % 8); the line's list entries are loaded 8 at a time (lane r holds entry
// p + r) and broadcast inside the 8-lane group, so a step is 3 shuffles, one 16-byte shared
// load and two RN multiply-adds.  List padding has value 0 (s + a 0 = s exactly for the
// finite nonnegative planes).  Chunk folds go straight to the output (first 1024-term chunk)
// or are added into it (later chunks).  pdl_tail: wait for the grid this one was launched
// beside before exiting, so stream successors are ordered after both.
__global__ void __maxnreg__(88)
    rad_quad_kernel(RadPair P, RadLists L, int nt1, int ngrp1, int nt2, int ngrp2, int pdl_tail) {
    extern __shared__ __align__(16) double rq_ds[];  // [RSUB][RQ_DL]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 3, r = lane & 7;
    const int K = (int)P.K;
    const int nsub = (K + RSUB - 1) / RSUB;
    const bool cen = !P.cflag || *P.cflag;  // uncentred planes (scan-written) unless flagged
    const bool on1 = rad_variant(P.mw1, P.M, P.K, P.N, 1) == 0, on2 = rad_variant(P.mw2, P.M, P.K, P.N, 0) == 1;
    const int n1 = nt1 * ngrp1, nitems = n1 + nt2 * ngrp2;
    bool used = false;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
        const bool first = item < n1;
        if (first ? !on1 : !on2) continue;
        const int it = first ? item : item - n1;
        const int ngrp = first ? ngrp1 : ngrp2;
        const int t0 = (it / ngrp) * RQ_DL;
        const int base = (it % ngrp) * RQ_LINES + warp * (4 * RQ_QW) + g;  // + 4 q
        const int TD = (int)(first ? P.M : P.N);  // dense lines (the strip's dimension)
        const int LN = (int)(first ? P.N : P.M);  // sparse lines
        const double* dense = first ? P.da1 : P.db2;  // [K][TD]: |A| transposed / |B| + R_B
        const int* cnt = first ? L.cnt1 : L.cnt2;
        const int* idx = first ? L.idx1 : L.idx2;
        const double* val = first ? L.val1 : L.val2;
        uint32_t* rb = first ? P.r1b : P.r2b;
        int64_t* rf = first ? P.r1f : P.r2f;
        const int d0 = t0 + 2 * r;  // this lane's dense lines d0, d0 + 1
        int64_t cd[2] = {0, 0};
        if (cen) {
#pragma unroll
            for (int h = 0; h < 2; h++)
                if (d0 + h < TD) cd[h] = first ? P.ec1[d0 + h] : P.fc2[d0 + h];
        }
        double acc[RQ_QW][2];
        int pcur[RQ_QW];
#pragma unroll
        for (int q = 0; q < RQ_QW; q++) {
            acc[q][0] = acc[q][1] = 0.0;
            pcur[q] = 0;
        }
        for (int sc = 0; sc < nsub; sc++) {
            const int c0 = sc * RSUB;
            if (used) __syncthreads();  // the previous strip is fully consumed
            used = true;
            // this sub-chunk's list segments of the warp's 8 quads: end positions, then the first
            // 8 entries of each (all loads issued before the strip copy is waited for)
            int pe[RQ_QW], cl[RQ_QW];
            double cv[RQ_QW];
#pragma unroll
            for (int q = 0; q < RQ_QW; q++) pe[q] = base + 4 * q < LN ? cnt[sc * LN + base + 4 * q] : 0;
            if ((TD & 1) == 0) {  // strip sub-chunk by 16-byte async copies (zero-filled outside the planes)
                const int c2 = 2 * (threadIdx.x & 7);
                const double* src = dense + (int64_t)c0 * TD + t0 + c2;
                const bool cok = t0 + c2 < TD;
#pragma unroll
                for (int u = 0; u < RSUB / (RQ_T / 8); u++) {
                    const int row = (threadIdx.x >> 3) + (RQ_T / 8) * u;
                    const bool ok = cok && c0 + row < K;
                    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(rq_ds + row * RQ_DL + c2);
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                                 "l"(ok ? src + (int64_t)row * TD : dense), "r"(ok ? 16 : 0)
                                 : "memory");
                }
                asm volatile("cp.async.commit_group;" ::: "memory");
            } else {  // odd leading dimension: thread -> (row e / 16, column e % 16), 8 loads in flight
                const int col = threadIdx.x & 15;
                const bool cok = t0 + col < TD;
                const double* src = dense + (int64_t)c0 * TD + t0 + col;
#pragma unroll 1
                for (int e0 = threadIdx.x; e0 < RSUB * RQ_DL; e0 += 8 * RQ_T) {
                    double t[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int row = (e0 >> 4) + (RQ_T / 16) * u;  // (e0 + RQ_T u) / 16
                        t[u] = (cok && c0 + row < K) ? src[(int64_t)row * TD] : 0.0;
                    }
#pragma unroll
                    for (int u = 0; u < 8; u++) rq_ds[e0 + RQ_T * u] = t[u];
                }
            }
#pragma unroll
            for (int q = 0; q < RQ_QW; q++) {
                const int line = base + 4 * q;
                const bool in = pcur[q] + r < pe[q];
                cl[q] = in ? idx[(int64_t)line * K + pcur[q] + r] : c0;
                cv[q] = in ? val[(int64_t)line * K + pcur[q] + r] : 0.0;
            }
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncthreads();
            const bool fold = ((sc + 1) * RSUB) % RCH == 0 || sc + 1 == nsub;
            const bool later = (sc * RSUB) / RCH > 0;  // not the first 1024-term chunk
            const double* strip = rq_ds + 2 * r - (int64_t)c0 * RQ_DL;
#pragma unroll
            for (int q = 0; q < RQ_QW; q++) {
                const int line = base + 4 * q;
                const bool live = line < LN;
                const int pend = pe[q];
                int p = pcur[q];
                const int* li = idx + (int64_t)line * K;
                const double* lv = val + (int64_t)line * K;
                int rem = __reduce_max_sync(0xffffffffu, pend - p);
                int cle = cl[q];
                double cve = cv[q];
                double a0 = acc[q][0], a1 = acc[q][1];
                while (rem > 0) {
                    const bool more = p + 8 + r < pend;
                    const int nl = more ? li[p + 8 + r] : c0;  // next 8 entries while these are consumed
                    const double nv = more ? lv[p + 8 + r] : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int l = __shfl_sync(0xffffffffu, cle, u, 8);
                        const double v = __shfl_sync(0xffffffffu, cve, u, 8);
                        const double2 x = *reinterpret_cast<const double2*>(strip + l * RQ_DL);
                        a0 = __dadd_rn(a0, __dmul_rn(x.x, v));
                        a1 = __dadd_rn(a1, __dmul_rn(x.y, v));
                    }
                    p += 8;
                    rem -= 8;
                    cle = nl;
                    cve = nv;
                }
                pcur[q] = pend;
                if (fold) {
                    if (live) {
                        const int64_t cs = cen ? (first ? P.fc1[line] : P.ec2[line]) : 0;
#pragma unroll
                        for (int h = 0; h < 2; h++) {
                            const int d = d0 + h;
                            if (d < TD) {
                                const double a = h ? a1 : a0;
                                const int64_t o = first ? (int64_t)d * P.N + line : (int64_t)line * P.N + d;
                                Mag m = a != 0.0 ? rad_fold_mag(a, -cd[h] - cs) : mag_zero();
                                if (later) m = mag_add(mag_load(rb[o], rf[o]), m);
                                mag_store(m, &rb[o], &rf[o]);
                            }
                        }
                    }
                    a0 = a1 = 0.0;
                }
                acc[q][0] = a0;
                acc[q][1] = a1;
            }
        }
    }
    if (pdl_tail) griddep_wait();
}

// dense variants (stand down unless picked): blockIdx.z = product
#ifndef APB_RADG_MINB
#define APB_RADG_MINB 8  // 128 registers, 16 warps/SM: 2.5% faster than 4 at N=2048 (c2 runs the 2x2 kernel)
#endif
template <int PT>
APB_DEV void rad_gemm2_body(const RadPair& P) {
    if (blockIdx.z == 0)
        rad_gemm_body<PT>(P.da1, P.db1, P.M, P.N, P.K, P.ec1, P.fc1, P.r1b, P.r1f, 0, 1, P.mw1, blockIdx.x,
                          blockIdx.y, P.cflag);
    else
        rad_gemm_body<PT>(P.da2, P.db2, P.M, P.N, P.K, P.ec2, P.fc2, P.r2b, P.r2f, 0, 0, P.mw2, blockIdx.x,
                          blockIdx.y, P.cflag);
}
__global__ void __launch_bounds__(64, APB_RADG_MINB) rad_gemm2_kernel(RadPair P) { rad_gemm2_body<4>(P); }
// small products (fewer 32 x 32 tiles than ~4 per SM): 2 x 2 outputs per thread,
// 4x the warps for the same tiles (c2: rad products 73 us at ~2 warps per SM)
// (88 registers: two of its warps fit on each SM sub-partition beside the 3 x 112-register warps of a
// raw-epilogue band-GEMM CTA, and its 30 KB of shared memory in what that CTA leaves, so on small
// products the dense radius runs next to the GEMM instead of in front of it)
__global__ void __maxnreg__(88) rad_gemm2s_kernel(RadPair P) { rad_gemm2_body<2>(P); }
// tiles of both dense products below which the 2 x 2 variant runs
constexpr int64_t RAD_SMALL_TILES = 4 * 148;

// exact double planes of both sides in one launch: blocks [0, nA) A, the rest B
__global__ void fused_planes2_kernel(BallsView A, BallsView B, RadPair P, int64_t nA) {
    if (P.cflag && !*P.cflag) return;  // the scan's uncentred planes are exact
    const bool a = (int64_t)blockIdx.x < nA;
    const int64_t t = ((int64_t)blockIdx.x - (a ? 0 : nA)) * blockDim.x + threadIdx.x;
    const int64_t rows = a ? P.M : P.K, cols = a ? P.K : P.N;
    double v1 = 0.0, v2 = 0.0;
    if (t < rows * cols) {
        const BallsView& X = a ? A : B;
        const int64_t line = a ? t / cols : t % cols;  // A: row i; B: column j
        const Mag m1 = rad_operand(X, t, a ? 0 : 2);
        const Mag m2 = rad_operand(X, t, a ? 1 : 3);
        const int64_t c1 = a ? P.ec1[line] : P.fc1[line], c2 = a ? P.ec2[line] : P.fc2[line];
        if (m1.kind == 1) v1 = ldexp((double)m1.b, (int)(m1.f - 30 + c1));
        if (m2.kind == 1) v2 = ldexp((double)m2.b, (int)(m2.f - 30 + c2));
        if (a) {  // |A| plane stored transposed ([l][i]) for coalesced column-list products
            P.da1[(t % cols) * rows + t / cols] = v1;
            P.da2[t] = v2;
        } else {
            P.db1[t] = v1;
            P.db2[t] = v2;
        }
    }
}

__global__ void count_nonzero_kernel(const double* p, int64_t n, unsigned long long* cnt) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool nz = t < n && p[t] != 0.0;
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(cnt, (unsigned long long)__popc(m));
}

// C.rad = mag_add(C.rad, mag_add(r1, r2)) (src/matmul.cpp:512-513)
__global__ void rad_combine_kernel(BallsOut C, int64_t cnt, const uint32_t* r1b, const int64_t* r1f,
                                   const uint32_t* r2b, const int64_t* r2f) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    Mag r = mag_add(mag_load(r1b[t], r1f[t]), mag_load(r2b[t], r2f[t]));
    Mag c = mag_load(C.rad_man[t], C.rad_exp[t]);
    mag_store(mag_add(c, r), &C.rad_man[t], &C.rad_exp[t]);
}

// ------------------------------------------------------------ K8 complex
__global__ void ball_addsub_kernel(BallsView X, BallsView Y, int negate_y, int64_t cnt, int64_t prec,
                                   BallsOut O, int* status) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= cnt) return;
    GF a, b;
    gf_load(a, X, t);
    gf_load(b, Y, t);
    if (negate_y) {
        if (b.kind == APB_FINITE) b.neg = !b.neg;
        else if (b.kind == APB_PINF) b.kind = APB_NINF;
        else if (b.kind == APB_NINF) b.kind = APB_PINF;
    }
    Mag err = gf_add_round(a, a, b, prec, status);
    if (a.kind == APB_NAN) {
        gf_store(O, t, a, mag_inf(), status);
        return;
    }
    Mag r = mag_add(mag_add(mag_load(X.rad_man[t], X.rad_exp[t]), mag_load(Y.rad_man[t], Y.rad_exp[t])), err);
    gf_store(O, t, a, r, status);
}

// ----------------------------------------------------------------- host

template <class T>
T* ws_buf(int slot, size_t count, cudaStream_t st) {
    return (T*)workspace().scratch(st, count * sizeof(T), slot);
}

struct Scratch {
    // separate allocations owned here (the Workspace slot table is small)
    void* p[64] = {};
    size_t cap[64] = {};
    uint64_t gen = 0;  // bumped on every reallocation (captured graphs hold these pointers)
    void* get(int k, size_t bytes, cudaStream_t st) {
        if (cap[k] < bytes) {
            gen++;
            if (p[k]) {
                cudaStreamSynchronize(st);
                cudaFree(p[k]);
            }
            size_t c = bytes + bytes / 4 + 256;
            if (cudaMalloc(&p[k], c) != cudaSuccess) {
                p[k] = nullptr;
                cap[k] = 0;
                return nullptr;
            }
            cap[k] = c;
        }
        return p[k];
    }
};
Scratch& scratch() {
    static Scratch s;
    return s;
}
enum {
    S_RTOP, S_RBOT, S_CTOP, S_CBOT, S_SUM, S_APACK, S_BPACK, S_TW, S_TC, S_UNITS, S_ESC, S_FSC,
    S_WA, S_WB, S_GREEDY, S_DA, S_DB, S_CEN_E, S_CEN_F, S_R1B, S_R1F, S_R2B, S_R2F, S_MISC, S_CTOP2, S_CBOT2, S_LCNT, S_LIDX, S_LVAL, S_DA2, S_DB2, S_CEN_E2, S_CEN_F2, S_RW1, S_RW2, S_LCNT2, S_LIDX2, S_LVAL2, S_RW1T, S_RW1B, S_RW2T, S_RW2B, S_CW1T, S_CW1B, S_CW2T, S_CW2B, S_PARTA, S_PARTB
};
template <class T>
T* sbuf(int k, size_t count, cudaStream_t st) {
    return (T*)scratch().get(k, count * sizeof(T) + 16, st);
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// host-side trace of the launch sequence (APB_HOST_TRACE=1 prints per call)
struct HostTrace {
    bool on = std::getenv("APB_HOST_TRACE") != nullptr;
    std::chrono::steady_clock::time_point t0;
    char buf[1024];
    int n = 0;
    void start() {
        if (!on) return;
        t0 = std::chrono::steady_clock::now();
        n = 0;
    }
    void mark(const char* what) {
        if (!on || n > 900) return;
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        n += std::snprintf(buf + n, sizeof buf - n, " %s=%.1f", what, us);
    }
    void flush() {
        if (on) std::fprintf(stderr, "host trace (us):%s\n", buf);
    }
};
HostTrace& htrace() {
    static HostTrace h;
    return h;
}

void scan_cols(const BallsView& b, int64_t K, int64_t N, int64_t lo, int64_t hi, int64_t* ctop,
               int64_t* cbot, ScanSummary* sum, cudaStream_t st) {
    init_minmax_kernel<<<blocks_for(N, 256), 256, 0, st>>>(ctop, cbot, N);
    dim3 grid(blocks_for(N, 128), blocks_for(hi - lo, COL_CHUNK));
    if (hi > lo) scan_cols_kernel<<<grid, 128, 0, st>>>(b, K, N, lo, hi, ctop, cbot, sum);
    col_width_kernel<<<blocks_for(N, 256), 256, 0, st>>>(ctop, cbot, N, &sum->maxw_b);
    count_launch(3);
}

int classical(const apb_mat* A, const apb_mat* B, int64_t prec, apb_mat* C, cudaStream_t st) {
    stats().classical_calls++;
    apb_dot_index ix;
    ix.bdiv = B->cols;
    ix.x_off = 0;
    ix.xs1 = A->cols;
    ix.xs2 = 0;
    ix.xstep = 1;
    ix.y_off = 0;
    ix.ys1 = 0;
    ix.ys2 = 1;
    ix.ystep = B->cols;
    return dot_batch_launch(&A->b, &B->b, nullptr, 0, &ix, A->cols, A->rows * B->cols, prec,
                            APB_DOT_BALL, nullptr, &C->b, nullptr, nullptr, 0, st);
}

// basecase block: c_ij = dot_ball(&c_ij, false, A[i, lo:hi], 1, B[lo:hi, j], N, w, p)
int basecase(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi, int64_t prec, apb_mat* C,
             cudaStream_t st) {
    apb_dot_index ix;
    ix.bdiv = B->cols;
    ix.x_off = lo;
    ix.xs1 = A->cols;
    ix.xs2 = 0;
    ix.xstep = 1;
    ix.y_off = lo * B->cols;
    ix.ys1 = 0;
    ix.ys2 = 1;
    ix.ystep = B->cols;
    return dot_batch_launch(&A->b, &B->b, &C->b, 0, &ix, hi - lo, A->rows * B->cols, prec,
                            APB_DOT_BALL, nullptr, &C->b, nullptr, nullptr, 0, st);
}

struct Plan {
    std::vector<int64_t> steps;  // triples (lo, hi, basecase)
    bool special = false;
    int64_t maxw_a = 0, maxw_b = 0;  // whole-range widths (single block)
    int64_t prec_a = 0, prec_b = 0;
};

// K3 launch: midpoint windows, specials and entry precision into `sum` (no sync)
int plan_launch(const apb_mat* A, const apb_mat* B, ScanSummary* sum, cudaStream_t st) {
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int64_t* rtop = sbuf<int64_t>(S_RTOP, M, st);
    int64_t* rbot = sbuf<int64_t>(S_RBOT, M, st);
    int64_t* ctop = sbuf<int64_t>(S_CTOP, N, st);
    int64_t* cbot = sbuf<int64_t>(S_CBOT, N, st);
    if (!rtop || !rbot || !ctop || !cbot || !sum) return APB_ERR_CUDA;
    cudaMemsetAsync(sum, 0, sizeof(ScanSummary), st);
    scan_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, 0, K, rtop, rbot, sum);
    scan_cols(b, K, N, 0, K, ctop, cbot, sum, st);
    count_launch(1);
    return APB_OK;
}

// K3 finish (host, after the sync): plan_blocks (src/matmul.cpp:132-161)
int plan_finish(const apb_mat* A, const apb_mat* B, int64_t prec, const ScanSummary& hs, Plan& P,
                cudaStream_t st) {
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int rc;
    P.special = hs.special_a || hs.special_b;
    if (P.special) return APB_OK;
    P.maxw_a = hs.maxw_a;
    P.maxw_b = hs.maxw_b;
    P.prec_a = hs.prec_a;
    P.prec_b = hs.prec_b;
    int64_t pm = std::max<int64_t>(hs.prec_a, hs.prec_b);
    pm = std::min<int64_t>(prec, pm);
    const int64_t h = (5 * pm) / 4 + 192;
    std::vector<int64_t> raw;
    if (hs.maxw_a <= h && hs.maxw_b <= h) {
        raw = {0, K};  // every window fits: greedy takes all of [0,K)
    } else {
        longlong2* wA = sbuf<longlong2>(S_WA, (size_t)M * K, st);
        longlong2* wB = sbuf<longlong2>(S_WB, (size_t)N * K, st);
        int64_t* gout = sbuf<int64_t>(S_GREEDY, 2 * (size_t)K + 2, st);
        int* gn = sbuf<int>(S_MISC, 1, st);
        if (!wA || !wB || !gout || !gn) return APB_ERR_CUDA;
        entry_windows_kernel<<<blocks_for(M * K + K * N, 256), 256, 0, st>>>(a, b, M, K, N, wA, wB);
        const size_t shm = (size_t)(M + N) * sizeof(longlong2);
        if (shm > 200 * 1024) {
            set_error("matmul planner: M+N too large for the device greedy split");
            return APB_ERR_UNSUPPORTED;
        }
        cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        greedy_kernel<<<1, 1024, shm, st>>>(wA, wB, K, M, N, h, gout, gn);
        count_launch(2);
        int n = 0;
        cudaMemcpyAsync(&n, gn, sizeof(int), cudaMemcpyDeviceToHost, st);
        if ((rc = cuda_check(cudaStreamSynchronize(st), "greedy"))) return rc;
        raw.resize(2 * (size_t)n);
        cudaMemcpy(raw.data(), gout, sizeof(int64_t) * 2 * n, cudaMemcpyDeviceToHost);
    }
    const int64_t nraw = (int64_t)raw.size() / 2;
    for (int64_t idx = 0; idx < nraw; idx++) {
        int64_t lo = raw[2 * idx], hi = raw[2 * idx + 1];
        if (hi - lo < 30) {  // short block -> dot basecase extended to 30 (src/matmul.cpp:149-155)
            hi = std::min<int64_t>(lo + 30, K);
            while (idx + 1 < nraw && raw[2 * (idx + 1) + 1] <= hi) idx++;
            if (idx + 1 < nraw && raw[2 * (idx + 1)] < hi) raw[2 * (idx + 1)] = hi;
            P.steps.insert(P.steps.end(), {lo, hi, 1});
        } else {
            P.steps.insert(P.steps.end(), {lo, hi, 0});
        }
    }
    return APB_OK;
}

ScanSummary* pinned_summary() {
    static ScanSummary* h = nullptr;
    if (!h) cudaMallocHost(&h, sizeof(ScanSummary) + 8 * sizeof(long long));
    return h;
}

int plan(const apb_mat* A, const apb_mat* B, int64_t prec, Plan& P, cudaStream_t st) {
    ScanSummary* sum = sbuf<ScanSummary>(S_SUM, 1, st);
    int rc = plan_launch(A, B, sum, st);
    if (rc) return rc;
    ScanSummary* hs = pinned_summary();
    cudaMemcpyAsync(hs, sum, sizeof(ScanSummary), cudaMemcpyDeviceToHost, st);
    if ((rc = cuda_check(cudaStreamSynchronize(st), "matmul plan scan"))) return rc;
    return plan_finish(A, B, prec, *hs, P, st);
}

// slice count for an exact |value| < 2^H with balanced digits (headroom 2 bits)
inline int slices_for(int64_t H) { return (int)((H + 2 + 7) / 8); }

// unit table + diagonal groups for the slice GEMM
struct Units {
    std::vector<int4> units;
    std::vector<int> group_begin, group_d1;
};

Units make_units(int SA, int SB, int64_t K, int tiles) {
    Units U;
    const int ND = SA + SB - 1;
    const int64_t pmax = std::max<int64_t>(1, 65535 / std::max<int64_t>(K, 1));  // |D| < 2^30
    std::vector<int64_t> pairs_upto_quad;  // work per 4-diagonal quad
    const int NQ = (ND + 3) / 4;
    std::vector<int64_t> quad_work(NQ, 0);
    for (int d = 0; d < ND; d++) {
        const int slo = std::max(0, d - SB + 1), shi = std::min(d, SA - 1) + 1;
        quad_work[d / 4] += shi - slo;
    }
    // groups: enough CTAs to fill the 148 SMs, balanced by pair count
    int64_t total = 0;
    for (auto w : quad_work) total += w;
    int G = std::max(1, std::min(NQ, (148 + tiles - 1) / tiles));
    const int64_t target = (total + G - 1) / G;
    U.group_begin.push_back(0);
    int64_t acc = 0;
    int q = 0;
    for (int d = 0; d < ND; d++) {
        const int slo = std::max(0, d - SB + 1), shi = std::min(d, SA - 1) + 1;
        for (int s = slo; s < shi; s += (int)pmax) {
            const int e = (int)std::min<int64_t>(shi, s + pmax);
            int flags = (s == slo ? 1 : 0) | (e == shi ? 2 : 0);
            U.units.push_back(make_int4(d, s, e, flags));
        }
        if ((d & 3) == 3 || d == ND - 1) {
            acc += quad_work[q++];
            const bool last = d == ND - 1;
            if (last || acc >= target * (int64_t)U.group_d1.size() + target) {
                U.group_d1.push_back(d + 1);
                U.group_begin.push_back((int)U.units.size());
            }
        }
    }
    return U;
}

// band GEMM geometry of a block of inner width w
struct BandGeom {
    int bn, band_w, Mp, Np, Kp;
};
BandGeom band_geom(int64_t M, int64_t N, int64_t w) {
    // band tile: 128 x 256 outputs with 2 diagonals per pass (N=256 MMAs) when the
    // matrix is wide enough, else 128 x 128 with 4 diagonals (APB_BAND_BN overrides)
    static const int bn_env = std::getenv("APB_BAND_BN") ? std::atoi(std::getenv("APB_BAND_BN")) : 0;
    BandGeom g;
    g.bn = bn_env == 128 || bn_env == 256 ? bn_env : (N >= 256 ? 256 : 128);
    g.band_w = g.bn == 256 ? 2 : 4;
    g.Mp = (int)((M + kSliceTile - 1) / kSliceTile * kSliceTile);
    g.Np = (int)((N + g.bn - 1) / g.bn * g.bn);
    g.Kp = (int)((w + kSliceBK - 1) / kSliceBK * kSliceBK);
    return g;
}

// digit-word template (2, 5 or 8 words) of the byte-parallel pack for S slices; 0 = byte-serial
inline int pack_ncw(int S) { return S <= 16 ? 2 : S <= 40 ? 5 : S <= 64 ? 8 : S <= 72 ? 9 : 0; }

// radius products to fold into the recombine (single block): the recombine waits
// for `ready` (recorded by the radius stream) and stores C.rad = err (+) (r1 (+) r2)
struct RadFuse {
    const uint32_t* r1b;
    const int64_t* r1f;
    const uint32_t* r2b;
    const int64_t* r2f;
    cudaEvent_t ready;
    bool capturing;
    bool used;  // out: the recombine took the radius (no rad_combine_kernel needed)
    bool joined = false;  // the stream already waited for `ready` (before the GEMM): no second wait
};
void wait_event(cudaStream_t s, cudaEvent_t ev, bool capturing);

int scaled_block(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi, int64_t prec, apb_mat* C,
                 bool first, int64_t maxw_a, int64_t maxw_b, const int64_t* rtop_in,
                 const int64_t* rbot_in, const int64_t* ctop_in, const int64_t* cbot_in,
                 int64_t* int_out, int int_limbs, int64_t* esc_out, int64_t* fsc_out,
                 cudaStream_t st, const std::function<int()>* after_gemm = nullptr, bool prepacked = false,
                 RadFuse* fuse = nullptr, const long long* spec_maxw = nullptr) {
    const int64_t M = A->rows, K = A->cols, N = B->cols, w = hi - lo;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    const int64_t* rtop = rtop_in;
    const int64_t* rbot = rbot_in;
    const int64_t* ctop = ctop_in;
    const int64_t* cbot = cbot_in;
    if (!rtop) {  // windows of this block only
        int64_t* rt = sbuf<int64_t>(S_RTOP, M, st);
        int64_t* rb = sbuf<int64_t>(S_RBOT, M, st);
        int64_t* ct = sbuf<int64_t>(S_CTOP, N, st);
        int64_t* cb = sbuf<int64_t>(S_CBOT, N, st);
        ScanSummary* sum = sbuf<ScanSummary>(S_SUM, 1, st);
        cudaMemsetAsync(sum, 0, sizeof(ScanSummary), st);
        scan_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, lo, hi, rt, rb, sum);
        scan_cols(b, K, N, lo, hi, ct, cb, sum, st);
        count_launch(1);
        ScanSummary h;
        cudaMemcpyAsync(&h, sum, sizeof h, cudaMemcpyDeviceToHost, st);
        int rc = cuda_check(cudaStreamSynchronize(st), "block scan");
        if (rc) return rc;
        maxw_a = h.maxw_a;
        maxw_b = h.maxw_b;
        rtop = rt;
        rbot = rb;
        ctop = ct;
        cbot = cb;
    }
    const int SA = slices_for(maxw_a), SB = slices_for(maxw_b);
    const BandGeom geo = band_geom(M, N, w);
    const int Mp = geo.Mp, Np = geo.Np, Kp = geo.Kp;
    stats().int_gemm_products++;
    stats().last_height_a = (uint64_t)maxw_a;
    stats().last_height_b = (uint64_t)maxw_b;
    stats().last_slices_a = (uint64_t)SA;
    stats().last_slices_b = (uint64_t)SB;
    int8_t* Ap = sbuf<int8_t>(S_APACK, (size_t)SA * Mp * Kp, st);
    int8_t* Bp = sbuf<int8_t>(S_BPACK, (size_t)SB * Np * Kp, st);
    int64_t* esc = esc_out ? esc_out : sbuf<int64_t>(S_ESC, M, st);
    int64_t* fsc = fsc_out ? fsc_out : sbuf<int64_t>(S_FSC, N, st);
    if (!Ap || !Bp || !esc || !fsc) {  // (slice planes are rewritten in full by the pack kernels)
        set_error("out of device memory (slice planes)");
        return APB_ERR_CUDA;
    }
    int tok = prof_begin("pack", st);
    if (!prepacked) {
        // byte-parallel recoding for up to 64 digits, byte-serial streams beyond
        static const bool v1 = std::getenv("APB_PACK_V1") != nullptr;  // test hook
        const unsigned ga = blocks_for((int64_t)Mp * Kp, 256);
        const int ca = v1 ? 0 : (SA + 7) / 8;
        if (ca >= 1 && ca <= 2) pack_a_v2_kernel<2><<<ga, 256, 0, st>>>(a, M, K, lo, hi, rtop, rbot, SA, Mp, Kp, Ap, esc);
        else if (ca >= 3 && ca <= 5) pack_a_v2_kernel<5><<<ga, 256, 0, st>>>(a, M, K, lo, hi, rtop, rbot, SA, Mp, Kp, Ap, esc);
        else if (ca >= 6 && ca <= 8) pack_a_v2_kernel<8><<<ga, 256, 0, st>>>(a, M, K, lo, hi, rtop, rbot, SA, Mp, Kp, Ap, esc);
        else if (ca == 9) pack_a_v2_kernel<9><<<ga, 256, 0, st>>>(a, M, K, lo, hi, rtop, rbot, SA, Mp, Kp, Ap, esc);  // (config 4: 69 slices)
        else pack_kernel<false><<<blocks_for((int64_t)Mp * Kp / 4, 256), 256, 0, st>>>(a, M, K, lo, hi, rtop, rbot, SA, Mp, Kp, Ap, esc);
        dim3 gb((unsigned)(Np / 32), (unsigned)(Kp / 32));
        const int cb = v1 ? 0 : (SB + 7) / 8;
        if (cb >= 1 && cb <= 2) pack_b_v2_kernel<2><<<gb, 256, 0, st>>>(b, N, lo, hi, ctop, cbot, SB, Np, Kp, Bp, fsc);
        else if (cb >= 3 && cb <= 5) pack_b_v2_kernel<5><<<gb, 256, 0, st>>>(b, N, lo, hi, ctop, cbot, SB, Np, Kp, Bp, fsc);
        else if (cb >= 6 && cb <= 8) pack_b_v2_kernel<8><<<gb, 256, 0, st>>>(b, N, lo, hi, ctop, cbot, SB, Np, Kp, Bp, fsc);
        else if (cb == 9) pack_b_v2_kernel<9><<<gb, 256, 0, st>>>(b, N, lo, hi, ctop, cbot, SB, Np, Kp, Bp, fsc);
        else pack_b_tiled_kernel<<<gb, 256, 0, st>>>(b, N, lo, hi, ctop, cbot, SB, Np, Kp, Bp, fsc);
    }
    prof_end(tok, st);
    if (!prepacked) count_launch(2);
    htrace().mark("pack_launched");
    const int ND = SA + SB - 1;
    // band kernel when every diagonal fits an int32 accumulator: pairs * w * 2^14 < 2^31
    static const bool force_unit = std::getenv("APB_FORCE_UNIT_GEMM") != nullptr;  // test hook
    // (or, beyond that, with in-place normalisations of the accumulators every kb_norm
    // K blocks: pairs * 128 kb_norm < 2^17)
    const int64_t pairs = std::min(SA, SB);
    static const bool no_norm = std::getenv("APB_NO_BAND_NORM") != nullptr;  // test hook: unit GEMM instead
    const bool fits = pairs * w < (int64_t)1 << 17;
    static const int kb_force = std::getenv("APB_BAND_KBNORM") ? std::atoi(std::getenv("APB_BAND_KBNORM")) : 0;
    // per item on the device: min(kb_norm, (2^17 - 1) / (its pairs * 128)); 1 << 20 = "as needed"
    int kb_norm = fits ? 0 : (((int64_t)1 << 17) - 1) / (pairs * kSliceBK) >= 1 ? 1 << 20 : 0;
    if (kb_force > 0) kb_norm = kb_force;  // test hook: an event every kb_force K blocks
    const bool band = !force_unit && (fits || (!no_norm && kb_norm > 0));
    // the recombine that will read the planes: recombine16 takes the band GEMM's raw
    // accumulators (no epilogue arithmetic in the GEMM) when no normalisation is needed
    static const bool slow_rc = std::getenv("APB_SLOW_RECOMBINE") != nullptr;  // test hook
    static const bool r64_rc = std::getenv("APB_RECOMBINE64") != nullptr;      // test hook
    static const bool no_raw = std::getenv("APB_NO_RAW_EPI") != nullptr ||     // test hook: carry epilogue
                               std::getenv("APB_BAND_V2") != nullptr;         // (the v2 kernel has no raw mode)
    const bool raw_epi = band && first && !int_out && C && out_of(&C->b).mant && !slow_rc && !r64_rc && !no_raw &&
                         kb_norm == 0 && (ND + 1) / 2 <= 80;
    // raw mode always runs 2 diagonals per band (16-bit digits for recombine16); small products
    // that leave most SMs without a 128 x 256 item may take 128-wide tiles and split K between
    // CTAs (the raw planes of the splits are summed by the recombine): the (tile width, splits)
    // pair with the smallest LPT makespan in the cost model below wins
    const int band_w = raw_epi ? 2 : geo.band_w;
    int bn = geo.bn, ksplit = 1;
    const int n_kb_all = Kp / kSliceBK;
    auto band_weights = [&](std::vector<int64_t>& bw) {
        const int NB = (ND + band_w - 1) / band_w;
        bw.assign(NB, 0);
        for (int d = 0; d < ND; d++) bw[d / band_w] += std::min(d, SA - 1) - std::max(0, d - SB + 1) + 1;
    };
    // item cost in tensor-pipe clocks: MMAs of M=128, K=32 take 128 (N=256) / ~72 (N=128) clocks,
    // 4 per slice pair and K block, plus the item's epilogue (~8300 / ~4300 clocks for a 128 x 256 /
    // 128 x 128 tile, measured; the accumulators are single-buffered, so an epilogue is not hidden
    // behind the next item's MMAs) and ~2500 clocks to fill the pipeline
    auto item_cost = [&](int64_t pairs_b, int tile_n, int kbs) -> int64_t {
        return pairs_b * kbs * (tile_n == 256 ? 512 : 288) + (tile_n == 256 ? 8300 : 4300) + 700;
    };
    auto makespan = [&](int tile_n, int ks) -> int64_t {
        std::vector<int64_t> bw;
        band_weights(bw);
        const int kbs = (n_kb_all + ks - 1) / ks;
        std::vector<int64_t> it;
        const int nt = (Mp / kSliceTile) * (Np / tile_n);
        for (int t = 0; t < nt * ks; t++)
            for (int64_t x : bw) it.push_back(item_cost(x, tile_n, kbs));
        std::sort(it.begin(), it.end(), std::greater<int64_t>());
        std::vector<int64_t> load(std::min<size_t>(148, it.size()), 0);
        for (int64_t c : it) *std::min_element(load.begin(), load.end()) += c;
        return *std::max_element(load.begin(), load.end());
    };
    static const int bn_env = std::getenv("APB_BAND_BN") ? std::atoi(std::getenv("APB_BAND_BN")) : 0;
    static const int ks_env = std::getenv("APB_BAND_KSPLIT") ? std::atoi(std::getenv("APB_BAND_KSPLIT")) : 0;
    // (the model only matters while the 256-wide items are few; its answer is cached per shape)
    static std::map<std::vector<int64_t>, std::pair<int, int>> shape_cache;
    const std::vector<int64_t> shape_key = {SA, SB, Mp, Np, Kp};
    const bool many_items = Np % 256 == 0 && (int64_t)(Mp / kSliceTile) * (Np / 256) * ((ND + 1) / 2) >= 4 * 148;
    auto cached = shape_cache.find(shape_key);
    if (raw_epi && many_items && !bn_env && !ks_env) {
        bn = 256;
    } else if (raw_epi && cached != shape_cache.end()) {
        bn = cached->second.first;
        ksplit = cached->second.second;
    } else if (raw_epi) {
        int64_t best = INT64_MAX;
        for (int tn : {256, 128}) {
            if (Np % tn || (bn_env && tn != bn_env)) continue;
            for (int ks : {1, 2}) {
                if (ks > n_kb_all || (ks - 1) * ((n_kb_all + ks - 1) / ks) >= n_kb_all || (ks_env && ks != ks_env))
                    continue;  // (every split keeps at least one K block)
                if (ks > 1 && (int64_t)(Mp / kSliceTile) * (Np / tn) * ((ND + 1) / 2) >= 148) continue;  // enough items
                const int64_t m = makespan(tn, ks);
                if (m < best) {
                    best = m;
                    bn = tn;
                    ksplit = ks;
                }
            }
        }
        if (shape_cache.size() > 1024) shape_cache.clear();
        shape_cache[shape_key] = {bn, ksplit};
    }
    const int tiles = (Mp / kSliceTile) * (Np / bn);
    // work tables depend only on (band, S_A, S_B, w, tile grid): built once on the
    // host (LPT item assignment / unit groups), cached as device copies
    struct Tables {
        char* dev;
        int G, NW;
        size_t off_items, off_begin, off_d1, n_ctas;
    };
    static std::map<std::vector<int64_t>, Tables> table_cache;
    const std::vector<int64_t> key = {band ? bn : 0, SA, SB, w, Mp, Np, band_w, ksplit};
    auto hit = table_cache.find(key);
    if (hit == table_cache.end()) {
        Tables T{};
        std::vector<char> host;
        if (band) {
            const int NB = (ND + band_w - 1) / band_w;
            std::vector<int64_t> bw;
            band_weights(bw);
            std::vector<std::pair<int64_t, int2>> items;
            const int kbs = (n_kb_all + ksplit - 1) / ksplit;
            for (int t = 0; t < tiles; t++)
                for (int ks = 0; ks < ksplit; ks++)
                    for (int bnd = 0; bnd < NB; bnd++)
                        items.push_back({item_cost(bw[bnd], bn, std::min(kbs, n_kb_all - ks * kbs)), make_int2(t, bnd | (ks << 16))});
            std::stable_sort(items.begin(), items.end(),
                             [](const std::pair<int64_t, int2>& x, const std::pair<int64_t, int2>& y) {
                                 return x.first > y.first;
                             });
            T.n_ctas = std::min<size_t>(148, items.size());
            std::vector<std::vector<int2>> lists(T.n_ctas);
            std::vector<int64_t> load(T.n_ctas, 0);
            for (auto& it : items) {  // LPT: heaviest item to the least loaded CTA
                size_t best = 0;
                for (size_t c = 1; c < T.n_ctas; c++)
                    if (load[c] < load[best]) best = c;
                lists[best].push_back(it.second);
                load[best] += it.first;
            }
            std::vector<int2> flat;
            std::vector<int> begin = {0}, group_d1;
            for (auto& l : lists) {
                flat.insert(flat.end(), l.begin(), l.end());
                begin.push_back((int)flat.size());
            }
            for (int bnd = 0; bnd < NB; bnd++) group_d1.push_back(band_w * bnd + band_w);
            T.off_items = 0;
            T.off_begin = flat.size() * sizeof(int2);
            T.off_d1 = T.off_begin + begin.size() * sizeof(int);
            host.resize(T.off_d1 + group_d1.size() * sizeof(int));
            std::memcpy(host.data(), flat.data(), flat.size() * sizeof(int2));
            std::memcpy(host.data() + T.off_begin, begin.data(), begin.size() * sizeof(int));
            std::memcpy(host.data() + T.off_d1, group_d1.data(), group_d1.size() * sizeof(int));
            T.G = NB;
            T.NW = NB;
        } else {
            Units U = make_units(SA, SB, w, tiles);
            T.G = (int)U.group_d1.size();
            T.NW = (ND + 3) / 4;
            T.off_items = 0;
            T.off_begin = U.units.size() * sizeof(int4);
            T.off_d1 = T.off_begin + U.group_begin.size() * sizeof(int);
            host.resize(T.off_d1 + U.group_d1.size() * sizeof(int));
            std::memcpy(host.data(), U.units.data(), U.units.size() * sizeof(int4));
            std::memcpy(host.data() + T.off_begin, U.group_begin.data(), U.group_begin.size() * sizeof(int));
            std::memcpy(host.data() + T.off_d1, U.group_d1.data(), U.group_d1.size() * sizeof(int));
        }
        if (cudaMalloc(&T.dev, host.size()) != cudaSuccess) {
            set_error("out of device memory (unit tables)");
            return APB_ERR_CUDA;
        }
        cudaMemcpy(T.dev, host.data(), host.size(), cudaMemcpyHostToDevice);
        if (table_cache.size() > 256) {  // bounded cache
            cudaDeviceSynchronize();
            for (auto& kv : table_cache) cudaFree(kv.second.dev);
            table_cache.clear();
            scratch().gen++;  // device table pointers baked into captured graphs are gone
        }
        hit = table_cache.emplace(key, T).first;
    }
    const Tables& TB = hit->second;
    const int G = TB.G, NW = TB.NW;
    char* dunits = TB.dev;
    const size_t off_items = TB.off_items, off_begin = TB.off_begin, off_d1 = TB.off_d1, n_ctas = TB.n_ctas;
    uint32_t* Tw = sbuf<uint32_t>(S_TW, (size_t)NW * ksplit * Mp * Np, st);
    int32_t* Tc = sbuf<int32_t>(S_TC, (size_t)G * ksplit * Mp * Np, st);
    if (!Tw || !Tc) {
        set_error("out of device memory (product planes)");
        return APB_ERR_CUDA;
    }
    int rc;
    int raw_mode = 0;
    const int* d_group_d1 = (const int*)(dunits + off_d1);
    if (band) {
        BandGemmParams P;
        P.S_A = SA;
        P.S_B = SB;
        P.Mp = Mp;
        P.Np = Np;
        P.Kp = Kp;
        P.n_kb = Kp / kSliceBK;
        P.ND = ND;
        P.n_tiles_n = Np / bn;
        P.bn = bn;
        P.band_w = band_w;
        P.kb_norm = kb_norm;
        P.items = (const int2*)(dunits + off_items);
        P.cta_begin = (const int*)(dunits + off_begin);
        P.Tw = Tw;
        P.Tc = Tc;
        P.spec_maxw = spec_maxw;
        // 40-bit band values when |D0 + 256 D1| <= 257 pairs K 2^14 stays below 2^39
        static const bool no_v40 = std::getenv("APB_RAW32") != nullptr;  // test hook: two int32 planes
        raw_mode = !raw_epi ? 0 : (!no_v40 && pairs * w <= 130560) ? 2 : 1;
        P.raw = raw_mode;
        if (raw_epi && ksplit > 1) {
            P.n_bands = (ND + band_w - 1) / band_w;
            P.kb_per = (n_kb_all + ksplit - 1) / ksplit;
        }
        static const int dbg = std::getenv("APB_GEMM_DEBUG") ? std::atoi(std::getenv("APB_GEMM_DEBUG")) : 0;
        P.debug = dbg;  // timing experiments only (results are wrong when set)
        if (dbg & 4) {  // clock64 trace of the band kernel, dumped to stderr after the call
            static long long* ts = nullptr;
            if (!ts) cudaMalloc(&ts, 148 * 32 * sizeof(long long));
            cudaMemsetAsync(ts, 0, 148 * 32 * sizeof(long long), st);
            P.dbg_ts = ts;
        }
        rc = band_gemm_launch(Ap, Bp, P, (int)n_ctas, st);
        if (P.dbg_ts) {
            long long h[148 * 32];
            cudaMemcpy(h, P.dbg_ts, sizeof h, cudaMemcpyDeviceToHost);
            for (size_t c = 0; c < n_ctas; c++) {
                std::fprintf(stderr, "cta %zu:", c);
                const long long t0 = h[c * 32 + 31];
                for (int k = 0; k < 4; k++)
                    if (h[c * 32 + 8 * k])
                        std::fprintf(stderr, " [w%lld i%lld c%lld e%lld..%lld]", h[c * 32 + 8 * k] - t0,
                                     h[c * 32 + 8 * k + 1] - t0, h[c * 32 + 8 * k + 2] - t0, h[c * 32 + 8 * k + 3] - t0,
                                     h[c * 32 + 8 * k + 4] - t0);
                std::fprintf(stderr, "\n");
            }
        }
    } else {
        SliceGemmParams P;
        P.S_A = SA;
        P.S_B = SB;
        P.Mp = Mp;
        P.Np = Np;
        P.Kp = Kp;
        P.n_kb = Kp / kSliceBK;
        P.units = (const int4*)(dunits + off_items);
        P.group_unit_begin = (const int*)(dunits + off_begin);
        P.group_d1 = d_group_d1;
        P.Tw = Tw;
        P.Tc = Tc;
        rc = slice_gemm_launch(Ap, Bp, P, G, st);
    }
    if (rc) return rc;
    htrace().mark("gemm_launched");
    if (after_gemm && (rc = (*after_gemm)())) return rc;
    htrace().mark("hook_done");
    RecombineArgs R;
    R.Tw = Tw;
    R.Tc = Tc;
    R.group_d1 = d_group_d1;
    R.n_groups = G;
    R.nwords = NW;
    R.Mp = Mp;
    R.Np = Np;
    R.M = M;
    R.N = N;
    R.escale = esc;
    R.fscale = fsc;
    if (C) {
        R.C = out_of(&C->b);
    } else {
        std::memset(&R.C, 0, sizeof R.C);
    }
    R.first = first ? 1 : 0;
    R.prec = prec;
    R.int_out = int_out;
    R.int_limbs = int_limbs;
    R.status = workspace().status_dev;
    R.quad = band ? 1 : 0;
    R.digit_bits = band ? 8 * band_w : 32;
    R.raw = raw_mode;
    R.nsplit = ksplit;
    R.spec_maxw = spec_maxw;
    R.spec_sa = SA;
    R.spec_sb = SB;
    tok = prof_begin("recombine", st);
    {
        const int NT = (int)(((int64_t)R.digit_bits * NW + 63) / 64) + 2;
        const unsigned gb = blocks_for(M * N, 128);
        const unsigned gbq = blocks_for(M * ((N + 3) / 4) * 4, 128);
        static const bool slow = std::getenv("APB_SLOW_RECOMBINE") != nullptr;  // test hook
        static const bool r64 = std::getenv("APB_RECOMBINE64") != nullptr;      // test hook
        const bool fast = band && first && !int_out && R.C.mant && !slow;
        if (fuse) {
            fuse->used = fast && band_w == 2 && NW <= 80 && !r64;  // recombine16 below
            if (fuse->used) {
                if (!fuse->joined) wait_event(st, fuse->ready, fuse->capturing);
                R.r1b = fuse->r1b;
                R.r1f = fuse->r1f;
                R.r2b = fuse->r2b;
                R.r2f = fuse->r2f;
            }
        }
        // APB_RC_PDL=1: recombine16 as the raw-epilogue GEMM's programmatic dependent.  Measured at
        // config 3: its blocks wait beside the GEMM CTAs from the GEMM's start and slow it from 91.5 to
        // 97.4 us; the plain launch starts 0.1 us after the GEMM's end once no event wait sits between
        // the two (RadFuse::joined), so it is the default
        static const bool rc_pdl = std::getenv("APB_RC_PDL") && std::atoi(std::getenv("APB_RC_PDL")) == 1;
        auto rc16_launch = [&](auto kern) {
            if (rc_pdl && raw_mode && spec_maxw) launch_pdl(kern, dim3(gbq), dim3(128), 0, st, R);
            else kern<<<gbq, 128, 0, st>>>(R);
        };
        if (fast && band_w == 4 && NW <= 20) recombine_fast_kernel<20, 32><<<gbq, 128, 0, st>>>(R);
        else if (fast && band_w == 4 && NW <= 40) recombine_fast_kernel<40, 32><<<gbq, 128, 0, st>>>(R);
        else if (fast && band_w == 4 && NW <= 72) recombine_fast_kernel<72, 32><<<gbq, 128, 0, st>>>(R);
        else if (fast && band_w == 2 && NW <= 40 && !r64 && ksplit > 1 && raw_mode == 2) rc16_launch(recombine16_kernel<40, true, true>);
        else if (fast && band_w == 2 && NW <= 80 && !r64 && ksplit > 1 && raw_mode == 2) rc16_launch(recombine16_kernel<80, true, true>);
        else if (fast && band_w == 2 && NW <= 40 && !r64 && ksplit > 1) rc16_launch(recombine16_kernel<40, true>);
        else if (fast && band_w == 2 && NW <= 80 && !r64 && ksplit > 1) rc16_launch(recombine16_kernel<80, true>);
        else if (fast && band_w == 2 && NW <= 40 && !r64 && raw_mode == 2) rc16_launch(recombine16_kernel<40, false, true>);
        else if (fast && band_w == 2 && NW <= 80 && !r64 && raw_mode == 2) rc16_launch(recombine16_kernel<80, false, true>);
        else if (fast && band_w == 2 && NW <= 40 && !r64) rc16_launch(recombine16_kernel<40>);
        else if (fast && band_w == 2 && NW <= 80 && !r64) rc16_launch(recombine16_kernel<80>);
        else if (fast && band_w == 2 && NW <= 40) recombine_fast_kernel<40, 16><<<gbq, 128, 0, st>>>(R);
        else if (fast && band_w == 2 && NW <= 80) recombine_fast_kernel<80, 16><<<gbq, 128, 0, st>>>(R);
        else if (fast && band_w == 2 && NW <= 144) recombine_fast_kernel<144, 16><<<gbq, 128, 0, st>>>(R);
        else if (NT <= 8) recombine_kernel<8><<<gb, 128, 0, st>>>(R);
        else if (NT <= 16) recombine_kernel<16><<<gb, 128, 0, st>>>(R);
        else if (NT <= 40) recombine_kernel<40><<<gb, 128, 0, st>>>(R);
        else recombine_kernel<GCAP><<<gb, 128, 0, st>>>(R);
    }
    prof_end(tok, st);
    count_launch();
    return cuda_check(cudaGetLastError(), "recombine");
}

void rad_center_cols(const BallsView& b, int64_t K, int64_t N, int64_t lo, int64_t hi, int which,
                     int64_t* fcen, long long* maxw, cudaStream_t st) {
    int64_t* ct = sbuf<int64_t>(S_CTOP2, N, st);
    int64_t* cb = sbuf<int64_t>(S_CBOT2, N, st);
    init_minmax_kernel<<<blocks_for(N, 256), 256, 0, st>>>(ct, cb, N);
    dim3 grid(blocks_for(N, 128), blocks_for(hi - lo, COL_CHUNK));
    if (hi > lo) rad_cols_minmax_kernel<<<grid, 128, 0, st>>>(b, K, N, lo, hi, which, ct, cb);
    rad_cols_center_kernel<<<blocks_for(N, 256), 256, 0, st>>>(ct, cb, N, fcen, maxw);
    count_launch(3);
}

// radius_matmul_upper(P, Q) into (rb, rf) for operand kinds (wa of A, wb of B)
struct RadSlots {
    int da, db, ce, cf, mw, lcnt, lidx, lval;
};
const RadSlots kRad[2] = {{S_DA, S_DB, S_CEN_E, S_CEN_F, S_RW1, S_LCNT, S_LIDX, S_LVAL},
                          {S_DA2, S_DB2, S_CEN_E2, S_CEN_F2, S_RW2, S_LCNT2, S_LIDX2, S_LVAL2}};

// radius_matmul_upper phase 1 (no sync): single-block centring, exact double
// planes, window widths and nonzero counts into mw[0..3]
int radius_prepare(const apb_mat* A, const apb_mat* B, int wa, int wb, int slot, cudaStream_t st) {
    const RadSlots& R = kRad[slot];
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int64_t* ecen = sbuf<int64_t>(R.ce, M, st);
    int64_t* fcen = sbuf<int64_t>(R.cf, N, st);
    long long* mw = sbuf<long long>(R.mw, 4, st);
    double* da = sbuf<double>(R.da, (size_t)M * K, st);
    double* db = sbuf<double>(R.db, (size_t)K * N, st);
    if (!ecen || !fcen || !mw || !da || !db) return APB_ERR_CUDA;
    cudaMemsetAsync(mw, 0, 4 * sizeof(long long), st);
    rad_center_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, 0, K, wa, ecen, mw);
    rad_center_cols(b, K, N, 0, K, wb, fcen, mw + 1, st);
    rad_planes_kernel<<<blocks_for(M * K, 256), 256, 0, st>>>(a, M, K, 0, K, wa, 1, ecen, da);
    rad_planes_kernel<<<blocks_for(K * N, 256), 256, 0, st>>>(b, K, N, 0, K, wb, 0, fcen, db);
    count_nonzero_kernel<<<blocks_for(M * K, 256), 256, 0, st>>>(da, M * K, (unsigned long long*)(mw + 2));
    count_nonzero_kernel<<<blocks_for(K * N, 256), 256, 0, st>>>(db, K * N, (unsigned long long*)(mw + 3));
    count_launch(5);
    return APB_OK;
}

// phase 2, given hw = mw copied to the host: sparse / dense single block, or the
// multi-block greedy path (which synchronizes `st` itself)
int radius_compute(const apb_mat* A, const apb_mat* B, int wa, int wb, int slot, const long long* hw,
                   uint32_t* rb, int64_t* rf, cudaStream_t st, int a_trans = 0) {
    const RadSlots& R = kRad[slot];
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int64_t* ecen = sbuf<int64_t>(R.ce, M, st);
    int64_t* fcen = sbuf<int64_t>(R.cf, N, st);
    double* da = sbuf<double>(R.da, (size_t)M * K, st);
    double* db = sbuf<double>(R.db, (size_t)K * N, st);
    int rc;
    if (hw[0] <= 900 && hw[1] <= 900) {
        // sparse products when one radius side is mostly exact (config 3: 95% of entries)
        const double dens_a = M * K ? (double)hw[2] / (double)(M * K) : 1.0;
        const double dens_b = K * N ? (double)hw[3] / (double)(K * N) : 1.0;
        int* lcnt = sbuf<int>(R.lcnt, (size_t)std::max(M, N), st);
        int* lidx = sbuf<int>(R.lidx, (size_t)K * std::max(M, N), st);
        double* lval = sbuf<double>(R.lval, (size_t)K * std::max(M, N), st);
        const int tk = prof_begin("rad_gemm", st);
        static const bool v1 = std::getenv("APB_RAD_V1") != nullptr;  // test hook: list kernels
        static const bool v2 = std::getenv("APB_RAD_V2") != nullptr;  // test hook: one line per thread
        if (!v1 && a_trans && dens_b <= 0.25 && dens_b <= dens_a) {
            if (v2 || M <= 256) rad_spcol_v2_kernel<<<(unsigned)N, 256, 0, st>>>(da, db, M, N, K, ecen, fcen, rb, rf);
            else rad_spcol_v3_kernel<2><<<(unsigned)N, 256, 0, st>>>(da, db, M, N, K, ecen, fcen, rb, rf);
        } else if (!v1 && !a_trans && dens_a <= 0.25) {
            if (v2 || N <= 256) rad_sprow_v2_kernel<<<(unsigned)M, 256, 0, st>>>(da, db, M, N, K, ecen, fcen, rb, rf);
            else rad_sprow_v3_kernel<2><<<(unsigned)M, 256, 0, st>>>(da, db, M, N, K, ecen, fcen, rb, rf);
        } else if (a_trans && dens_b <= 0.25 && dens_b <= dens_a && lcnt && lidx && lval) {
            col_lists_kernel<<<blocks_for(N, 8), 256, 0, st>>>(db, K, N, lcnt, lidx, lval);
            dim3 grid(blocks_for(M, 32), blocks_for(N, 8));
            rad_spcol_kernel<<<grid, 256, 0, st>>>(da, M, N, K, lcnt, lidx, lval, ecen, fcen, rb, rf);
        } else if (dens_a <= 0.25 && lcnt && lidx && lval) {
            row_lists_kernel<<<blocks_for(M, 8), 256, 0, st>>>(da, M, K, lcnt, lidx, lval, a_trans);
            dim3 grid(blocks_for(N, 256), (unsigned)M);
            rad_sprow_kernel<<<grid, 256, 0, st>>>(db, M, N, K, lcnt, lidx, lval, ecen, fcen, rb, rf);
        } else {
            dim3 grid(blocks_for(N, RT), blocks_for(M, RT));
            rad_gemm_kernel<<<grid, RTHREADS, 0, st>>>(da, db, M, N, K, ecen, fcen, rb, rf, 0, a_trans);
        }
        prof_end(tk, st);
        count_launch(2);
        return cuda_check(cudaGetLastError(), "radius product");
    }
    // greedy split with h = 900 on the Mag windows (f, f-30) (src/matmul.cpp:386-392)
    std::vector<int64_t> blocks;
    {
        longlong2* wA = sbuf<longlong2>(S_WA, (size_t)M * K, st);
        longlong2* wB = sbuf<longlong2>(S_WB, (size_t)N * K, st);
        int64_t* gout = sbuf<int64_t>(S_GREEDY, 2 * (size_t)K + 2, st);
        int* gn = sbuf<int>(S_MISC, 1, st);
        if (!wA || !wB || !gout || !gn) return APB_ERR_CUDA;
        mag_entry_windows_kernel<<<blocks_for(M * K + K * N, 256), 256, 0, st>>>(a, b, M, K, N, wa, wb, wA, wB);
        const size_t shm = (size_t)(M + N) * sizeof(longlong2);
        if (shm > 200 * 1024) {
            set_error("radius product: M+N too large for the device greedy split");
            return APB_ERR_UNSUPPORTED;
        }
        cudaFuncSetAttribute(greedy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        greedy_kernel<<<1, 1024, shm, st>>>(wA, wB, K, M, N, 900, gout, gn);
        count_launch(2);
        int n = 0;
        cudaMemcpyAsync(&n, gn, sizeof(int), cudaMemcpyDeviceToHost, st);
        if ((rc = cuda_check(cudaStreamSynchronize(st), "radius greedy"))) return rc;
        blocks.resize(2 * (size_t)n);
        cudaMemcpy(blocks.data(), gout, sizeof(int64_t) * 2 * n, cudaMemcpyDeviceToHost);
    }
    for (size_t bi = 0; bi + 1 < blocks.size(); bi += 2) {
        const int64_t lo = blocks[bi], hi = blocks[bi + 1], w = hi - lo;
        // centring over this block only
        rad_center_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, lo, hi, wa, ecen, nullptr);
        rad_center_cols(b, K, N, lo, hi, wb, fcen, nullptr, st);
        count_launch(1);
        rad_planes_kernel<<<blocks_for(M * w, 256), 256, 0, st>>>(a, M, K, lo, hi, wa, 1, ecen, da);
        rad_planes_kernel<<<blocks_for(w * N, 256), 256, 0, st>>>(b, K, N, lo, hi, wb, 0, fcen, db);
        dim3 grid(blocks_for(N, RT), blocks_for(M, RT));
        const int tk = prof_begin("rad_gemm", st);
        rad_gemm_kernel<<<grid, RTHREADS, 0, st>>>(da, db, M, N, w, ecen, fcen, rb, rf, bi ? 1 : 0, 0);
        prof_end(tk, st);
        count_launch(3);
    }
    return cuda_check(cudaGetLastError(), "radius product");
}

// radius_matmul_upper(P, Q) for operand kinds (wa of A, wb of B), synchronous planning
int radius_product(const apb_mat* A, const apb_mat* B, int wa, int wb, uint32_t* rb, int64_t* rf,
                   cudaStream_t st) {
    int rc = radius_prepare(A, B, wa, wb, 0, st);
    if (rc) return rc;
    long long* hw = (long long*)(pinned_summary() + 1);
    cudaMemcpyAsync(hw, sbuf<long long>(kRad[0].mw, 4, st), 4 * sizeof(long long), cudaMemcpyDeviceToHost, st);
    if ((rc = cuda_check(cudaStreamSynchronize(st), "radius windows"))) return rc;
    long long h[4] = {hw[0], hw[1], hw[2], hw[3]};
    return radius_compute(A, B, wa, wb, 0, h, rb, rf, st);
}

cudaStream_t side_stream() {
    static cudaStream_t s = [] {
        cudaStream_t t;
        cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
        return t;
    }();
    return s;
}

// ---- CUDA graphs for the launch sequence of block_matmul.  The fast path is
// three graphs per (operand pointers, shapes, precision, scratch generation):
//   G1 (main stream)  scan + finish, summary copy to pinned memory [event
//                     ev_plan], speculative slice pack;  [event ev_fin after the
//                     finish kernel]
//   GR (side stream)  radius planes + speculative products [event ev_join]
//   G2 (main stream)  band GEMM + recombine, wait ev_join, radius combine
// (G2 additionally keyed by the slice counts).  The host waits on ev_plan,
// plans, and launches G2 only when the speculation held (single block, slice
// counts within the packed template, single radius block, no specials);
// otherwise the eager path below runs, exactly as without graphs.  A call that
// misses the cache runs eagerly and captures the graphs for the next call.
struct GraphSet {
    cudaGraphExec_t g1 = nullptr, gr = nullptr;
    int64_t n1 = 0, nr = 0;  // kernels per launch (launch counter)
    // the whole single-block step as one graph (scan .. recombine, radius branch),
    // the GEMM and recombine speculating on the slice counts k2s of the last call
    std::map<std::vector<int64_t>, std::pair<cudaGraphExec_t, int64_t>> g1s;
    std::vector<int64_t> k2s;  // slice counts of the last call's plan
    std::map<std::vector<int64_t>, std::pair<cudaGraphExec_t, int64_t>> g2;
};

struct GraphCache {
    std::map<std::vector<int64_t>, GraphSet> sets;
    cudaStream_t cap = nullptr;
    cudaStream_t capture_stream() {
        if (!cap) cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
        return cap;
    }
    void clear() {
        cudaDeviceSynchronize();
        for (auto& kv : sets) {
            if (kv.second.g1) cudaGraphExecDestroy(kv.second.g1);
            for (auto& g : kv.second.g1s) cudaGraphExecDestroy(g.second.first);
            if (kv.second.gr) cudaGraphExecDestroy(kv.second.gr);
            for (auto& g : kv.second.g2) cudaGraphExecDestroy(g.second.first);
        }
        sets.clear();
    }
};
GraphCache& graphs() {
    static GraphCache g;
    return g;
}

// capture fn(stream) into an executable graph; returns nullptr on any failure
template <class F>
cudaGraphExec_t capture(F&& fn, int64_t* kernels) {
    cudaStream_t cs = graphs().capture_stream();
    const uint64_t before = apb_launch_count();
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    const int rc = fn(cs);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &g);
    const int64_t launched = (int64_t)(apb_launch_count() - before);
    launch_count_adjust(-launched);  // nothing ran; replays add the count
    *kernels = launched;
    cudaGraphExec_t ex = nullptr;
    if (rc == APB_OK && e == cudaSuccess && g && cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) ex = nullptr;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return ex;
}

void rec_event(cudaEvent_t ev, cudaStream_t s, bool capturing) {
    if (capturing) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
    else cudaEventRecord(ev, s);
}
void wait_event(cudaStream_t s, cudaEvent_t ev, bool capturing) {
    cudaStreamWaitEvent(s, ev, capturing ? cudaEventWaitExternal : 0);
}

cudaEvent_t make_event() {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    return e;
}

// the tiled sparse radius products: standalone (one CTA per item), or beside the band GEMM
// (pdl: launched as the GEMM's programmatic dependent on the GEMM's stream with at most one
// CTA per SM -- each fits next to a GEMM CTA -- and a tail wait for the GEMM grid)
struct RadDefer {
    RadPair rp;
    RadLists rl;
    bool ready = false;
};
int rad_quad_launch(const RadPair& rp, const RadLists& rl, cudaStream_t ss, bool pdl) {
    static const bool attr = [] {
        cudaFuncSetAttribute(rad_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, RQ_SMEM);
        cudaFuncSetAttribute(rad_quad_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        return true;
    }();
    (void)attr;
    const int nt1 = (int)blocks_for(rp.M, RQ_DL), ngrp1 = (int)blocks_for(rp.N, RQ_LINES);
    const int nt2 = (int)blocks_for(rp.N, RQ_DL), ngrp2 = (int)blocks_for(rp.M, RQ_LINES);
    const int64_t nitems = (int64_t)nt1 * ngrp1 + (int64_t)nt2 * ngrp2;
    cudaLaunchConfig_t cfg = {};
    static const int grid_force = std::getenv("APB_RAD_GRID") ? std::atoi(std::getenv("APB_RAD_GRID")) : 0;  // timing hook
    cfg.gridDim = dim3((unsigned)std::min<int64_t>(nitems, grid_force > 0 ? grid_force : pdl ? 148 : 148 * 7 * 2));
    cfg.blockDim = dim3(RQ_T);
    cfg.dynamicSmemBytes = RQ_SMEM;
    cfg.stream = ss;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
    cudaLaunchKernelEx(&cfg, rad_quad_kernel, rp, rl, nt1, ngrp1, nt2, ngrp2, pdl ? 1 : 0);
    return cuda_check(cudaGetLastError(), "radius products");
}

int block_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, apb_mat* C, cudaStream_t st) {
    // one host synchronisation: fused scans of A and B (planner windows and both
    // radius products' windows), centring, exact double planes and nonzero counts
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView av = view_of(&A->b), bv = view_of(&B->b);
    htrace().start();
    ScanSummary* sum = sbuf<ScanSummary>(S_SUM, 1, st);
    LineWins RW, CW;
    const int rslot[6] = {S_RTOP, S_RBOT, S_RW1T, S_RW1B, S_RW2T, S_RW2B};
    const int cslot[6] = {S_CTOP, S_CBOT, S_CW1T, S_CW1B, S_CW2T, S_CW2B};
    for (int q = 0; q < 3; q++) {
        RW.top[q] = sbuf<int64_t>(rslot[2 * q], M, st);
        RW.bot[q] = sbuf<int64_t>(rslot[2 * q + 1], M, st);
        CW.top[q] = sbuf<int64_t>(cslot[2 * q], N, st);
        CW.bot[q] = sbuf<int64_t>(cslot[2 * q + 1], N, st);
    }
    // the radius windows ride in the summary: one D2H for the planner
    long long* mw1 = sum ? sum->mw : nullptr;
    long long* mw2 = sum ? sum->mw + 4 : nullptr;
    int64_t* ec1 = sbuf<int64_t>(kRad[0].ce, M, st);
    int64_t* ec2 = sbuf<int64_t>(kRad[1].ce, M, st);
    int64_t* fc1 = sbuf<int64_t>(kRad[0].cf, N, st);
    int64_t* fc2 = sbuf<int64_t>(kRad[1].cf, N, st);
    double* da1 = sbuf<double>(kRad[0].da, (size_t)M * K, st);
    double* db1 = sbuf<double>(kRad[0].db, (size_t)K * N, st);
    double* da2 = sbuf<double>(kRad[1].da, (size_t)M * K, st);
    double* db2 = sbuf<double>(kRad[1].db, (size_t)K * N, st);
    uint32_t* r1b = sbuf<uint32_t>(S_R1B, (size_t)M * N, st);
    int64_t* r1f = sbuf<int64_t>(S_R1F, (size_t)M * N, st);
    uint32_t* r2b = sbuf<uint32_t>(S_R2B, (size_t)M * N, st);
    int64_t* r2f = sbuf<int64_t>(S_R2F, (size_t)M * N, st);
    const int cA = (int)((K + SCAN_A_COLS - 1) / SCAN_A_COLS), cB = (int)((K + SCAN_B_ROWS - 1) / SCAN_B_ROWS);
    int64_t* pa = sbuf<int64_t>(S_PARTA, (size_t)SCAN_FIELDS * cA * M, st);
    int64_t* pb = sbuf<int64_t>(S_PARTB, (size_t)SCAN_FIELDS * cB * N, st);
    if (!sum || !mw1 || !mw2 || !ec1 || !ec2 || !fc1 || !fc2 || !da1 || !db1 || !da2 || !db2 || !r1b || !r1f ||
        !r2b || !r2f || !pa || !pb)
        return APB_ERR_CUDA;
    // where the radius products run: 0 side stream after planning, 1 main stream
    // after the midpoint product, 2 side stream issued right after the GEMM
    // launch, 3 main stream before the midpoint product, 4 (default) side stream
    // right after the scan, before the host round trip -- speculatively assuming
    // a single radius block, with the sparse/dense kernel chosen on the device;
    // the multi-block case is redone on the main stream after the plan is known
    static const int rad_order = std::getenv("APB_RAD_ORDER") ? std::atoi(std::getenv("APB_RAD_ORDER")) : 4;
    static const bool no_spec_pack = std::getenv("APB_NO_SPEC_PACK") != nullptr;  // test hook
    static const bool no_graphs = std::getenv("APB_NO_GRAPHS") != nullptr;        // test hook
    static cudaEvent_t ev_join = make_event(), ev_fin = make_event(), ev_plan = make_event();
    static cudaEvent_t ev_fork = make_event(), ev_cjoin = make_event();
    static cudaStream_t cps = [] {
        cudaStream_t t;
        cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
        return t;
    }();
    static cudaStream_t pks = [] {  // the early pack's branch
        cudaStream_t t;
        cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
        return t;
    }();
    static cudaEvent_t ev_scan = make_event(), ev_packed1 = make_event();
    const bool spec = rad_order == 4;
    // speculative slice packing for the single-block plan of (almost) every
    // input, issued before the host round trip: the slice counts come from the
    // scan on the device (the kernels stand down if they exceed the template);
    // the host re-packs after planning when the guess does not hold
    const BandGeom sgeo = band_geom(M, N, K);
    const int guess_s = slices_for(std::max<int64_t>(prec, 2) + 8);
    const int sncw = no_spec_pack ? 0 : pack_ncw(guess_s);
    int8_t* sAp = nullptr;
    int8_t* sBp = nullptr;
    int64_t* esc = nullptr;
    int64_t* fsc = nullptr;
    if (sncw) {
        sAp = sbuf<int8_t>(S_APACK, (size_t)8 * sncw * sgeo.Mp * sgeo.Kp, st);
        sBp = sbuf<int8_t>(S_BPACK, (size_t)8 * sncw * sgeo.Np * sgeo.Kp, st);
        esc = sbuf<int64_t>(S_ESC, M, st);
        fsc = sbuf<int64_t>(S_FSC, N, st);
        if (!sAp || !sBp || !esc || !fsc) return APB_ERR_CUDA;
    }
    ScanSummary* hs = pinned_summary();
    long long* hw = hs->mw;

    // early pack: the speculative pack only needs the scan (line windows from the chunk partials,
    // every template plane written), so it runs on its own branch right behind the scan, beside
    // the finish kernel, instead of after it (APB_NO_EARLY_PACK=1: behind the finish kernel)
    static const bool no_early = std::getenv("APB_NO_EARLY_PACK") != nullptr;
    const bool early_ok = sncw && !no_early && !prof_enabled();
    // (Sa, Sb): planes the early pack writes -- the speculated slice counts in the fused step's graph
    // (a product that needs more is re-packed by the host), else all template planes
    auto launch_pack = [&](cudaStream_t ps, bool from_partials, int Sa = 0, int Sb = 0) {
        PackAB pk;
        pk.a = av;
        pk.b = bv;
        pk.M = M;
        pk.K = K;
        pk.N = N;
        pk.rtop = RW.top[0];
        pk.rbot = RW.bot[0];
        pk.ctop = CW.top[0];
        pk.cbot = CW.bot[0];
        pk.Mp = sgeo.Mp;
        pk.Np = sgeo.Np;
        pk.Kp = sgeo.Kp;
        pk.Ap = sAp;
        pk.Bp = sBp;
        pk.esc = esc;
        pk.fsc = fsc;
        pk.mwa = &sum->maxw_a;
        pk.mwb = &sum->maxw_b;
        if (from_partials) {
            pk.pa = pa;
            pk.pb = pb;
            pk.cA = cA;
            pk.cB = cB;
            pk.planes_a = Sa;
            pk.planes_b = Sb;
        }
        static const bool no_a4 = std::getenv("APB_PACK_A1") != nullptr;  // test hook: one entry per thread
        pk.a4 = no_a4 ? 0 : 1;
        pk.ga = blocks_for((int64_t)sgeo.Mp * sgeo.Kp / (pk.a4 ? 4 : 1), 256);
        pk.gbx = sgeo.Np / 32;
        const dim3 g((unsigned)(pk.ga + pk.gbx * (sgeo.Kp / 32)));
        // plain launch (not PDL): early-resident pack blocks waiting on the scan
        // would hold the SMs the radius products need right after it
        static const bool pack_pdl = std::getenv("APB_PACK_PDL") != nullptr;
        auto lp = [&](auto kern) {
            if (pack_pdl && !from_partials) launch_pdl(kern, g, dim3(256), 0, ps, pk);
            else kern<<<g, 256, 0, ps>>>(pk);
        };
        if (sncw == 2) lp(pack_ab_v2_kernel<2>);
        else if (sncw == 5) lp(pack_ab_v2_kernel<5>);
        else if (sncw == 9) lp(pack_ab_v2_kernel<9>);
        else lp(pack_ab_v2_kernel<8>);
        count_launch(1);
    };
    // `mid` (optional): work enqueued on `s` between the scan and the pack
    auto phase1 = [&](cudaStream_t s, bool capturing, const std::function<int(cudaStream_t)>* mid = nullptr,
                      int Sa = 0, int Sb = 0) -> int {
        const bool early = early_ok && !mid;
        const int tk_scan = prof_begin("scan", s);
        const int64_t nblk = M * cA + ((N + 31) / 32) * cB;
        static const bool no_scan_planes = std::getenv("APB_NO_SCAN_PLANES") != nullptr;  // test hook
        if (no_scan_planes)
            scan_v2_kernel<<<(unsigned)nblk, 256, 0, s>>>(av, bv, M, K, N, cA, cB, pa, pb, sum, mw1, mw2);
        else
            scan_v2_kernel<<<(unsigned)nblk, 256, 0, s>>>(av, bv, M, K, N, cA, cB, pa, pb, sum, mw1, mw2, da1, da2,
                                                          db1, db2);
        if (early) {
            cudaEventRecord(ev_scan, s);
            {  // launched before the pack, at the highest priority: its few blocks go ahead of the pack's
                static const int prio = [] {
                    int least = 0, greatest = 0;
                    cudaDeviceGetStreamPriorityRange(&least, &greatest);
                    return greatest;
                }();
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(blocks_for(32 * (M + N), 256));
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributePriority;
                at[0].val.priority = prio;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, scan_v2_finish_kernel, (const int64_t*)pa, (const int64_t*)pb, M, N, cA, cB,
                                   RW.top[0], RW.bot[0], CW.top[0], CW.bot[0], ec1, ec2, fc1, fc2, sum, mw1, mw2);
            }
            cudaStreamWaitEvent(pks, ev_scan, 0);
            launch_pack(pks, true, Sa, Sb);
            cudaEventRecord(ev_packed1, pks);
        } else {
            launch_pdl(scan_v2_finish_kernel, dim3(blocks_for(32 * (M + N), 256)), dim3(256), 0, s, pa, pb, M, N, cA,
                       cB, RW.top[0], RW.bot[0], CW.top[0], CW.bot[0], ec1, ec2, fc1, fc2, sum, mw1, mw2);
        }
        count_launch(2);
        prof_end(tk_scan, s);
        rec_event(ev_fin, s, capturing);
        // the planner summary leaves on a copy stream so the pack follows the scan directly
        cudaEventRecord(ev_fork, s);
        cudaStreamWaitEvent(cps, ev_fork, 0);
        cudaMemcpyAsync(hs, sum, sizeof(ScanSummary), cudaMemcpyDeviceToHost, cps);
        rec_event(ev_plan, cps, capturing);
        if (mid) {
            const int r = (*mid)(s);
            if (r) return r;
        }
        if (sncw && !early) {
            const int tk = prof_begin("pack", s);
            launch_pack(s, false);
            prof_end(tk, s);
        }
        if (early) cudaStreamWaitEvent(s, ev_packed1, 0);  // everything after phase 1 sees the slice planes
        cudaEventRecord(ev_cjoin, cps);
        cudaStreamWaitEvent(s, ev_cjoin, 0);
        return cuda_check(cudaGetLastError(), "matmul scan");
    };
    // speculative radius products (single radius block; sparse/dense chosen on the device)
    // `mid` (optional): a wait enqueued between the planes and the products
    // `which`: 1 sparse kernels, 2 dense kernels, 3 both (each stands down on the device unless picked)
    // centred planes in the speculative radius branch: when the previous product's operand
    // exponents were too far out for the scan's uncentred planes (config 4: radii near 2^-531),
    // this one most likely needs them too, so fused_planes2_kernel joins the branch (it stands
    // down on the device when the planes are fine) and the products are right the first time --
    // otherwise they would run on invalid planes and the host would redo the radius after the
    // midpoint product (at config 4: 0.45 ms wasted + 0.68 ms redone per real product)
    static std::map<std::vector<int64_t>, bool> want_planes_of;  // per (M, K, N, prec); under the API lock
    if (want_planes_of.size() > 4096) want_planes_of.clear();
    bool& want_planes = want_planes_of[{M, K, N, prec}];
    const bool planes_used = want_planes;
    auto phaseR = [&](cudaStream_t ss, bool capturing, cudaEvent_t mid = nullptr, RadDefer* defer = nullptr,
                      int which = 3) -> int {
        const int tk = prof_begin("radius", ss);
        static const bool no_scan_planes = std::getenv("APB_NO_SCAN_PLANES") != nullptr;
        RadPair rp{M, K, N, da1, db1, da2, db2, ec1, fc1, ec2, fc2, r1b, r2b, r1f, r2f, mw1, mw2,
                   no_scan_planes ? nullptr : &sum->rad_centred};
        static const bool split = std::getenv("APB_RAD_SPLIT") != nullptr;  // previous 6-launch schedule
        if (!split) {
            const int64_t nA = blocks_for(M * K, 256);
            if (no_scan_planes || planes_used)  // else the scan wrote uncentred planes (host redoes if flagged)
                fused_planes2_kernel<<<(unsigned)(nA + blocks_for(K * N, 256)), 256, 0, ss>>>(av, bv, rp, nA);
            if (mid) cudaStreamWaitEvent(ss, mid, 0);
            if (which & 1) {  // highest priority: its blocks are dispatched ahead of the pack's
                static const int prio = [] {
                    int least = 0, greatest = 0;
                    cudaDeviceGetStreamPriorityRange(&least, &greatest);
                    return std::getenv("APB_NO_PRIO") ? least : greatest;
                }();
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3((unsigned)(N + M));
                cfg.blockDim = dim3(256);
                cfg.stream = ss;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributePriority;
                at[0].val.priority = prio;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                // default: the per-line gather kernel (rad_sparse2); APB_RAD_QUAD=1: list
                // compaction + strip products (rad_lists + rad_quad), measured slower at
                // config 3 (6 + 23 us against 25 us, profiles/r2/radius_variants.txt)
                static const bool gather = std::getenv("APB_RAD_QUAD") == nullptr;
                const int64_t LNmax = std::max(M, N), nch = (K + RSUB - 1) / RSUB;
                RadLists rl{};
                if (!gather) {
                    rl.cnt1 = sbuf<int>(kRad[0].lcnt, (size_t)nch * LNmax, ss);
                    rl.idx1 = sbuf<int>(kRad[0].lidx, (size_t)K * LNmax, ss);
                    rl.val1 = sbuf<double>(kRad[0].lval, (size_t)K * LNmax, ss);
                    rl.cnt2 = sbuf<int>(kRad[1].lcnt, (size_t)nch * LNmax, ss);
                    rl.idx2 = sbuf<int>(kRad[1].lidx, (size_t)K * LNmax, ss);
                    rl.val2 = sbuf<double>(kRad[1].lval, (size_t)K * LNmax, ss);
                }
                if (!gather && rl.cnt1 && rl.idx1 && rl.val1 && rl.cnt2 && rl.idx2 && rl.val2) {
                    cfg.gridDim = dim3(blocks_for(32 * (N + M), 256));
                    cudaLaunchKernelEx(&cfg, rad_lists_kernel, rp, rl);
                    if (defer) {  // the caller launches the products beside the GEMM
                        defer->rp = rp;
                        defer->rl = rl;
                        defer->ready = true;
                    } else {
                        rad_quad_launch(rp, rl, ss, false);
                    }
                    count_launch(1);
                } else {
                    cudaLaunchKernelEx(&cfg, rad_sparse2_kernel<2, 256>, rp);
                }
            }
            if (which & 2) {
                const dim3 g2(blocks_for(N, RT), blocks_for(M, RT), 2);
                static const bool no_small = std::getenv("APB_RAD_NO_SMALL") != nullptr;  // test hook
                if (!no_small && (int64_t)g2.x * g2.y * 2 < RAD_SMALL_TILES)
                    rad_gemm2s_kernel<<<g2, 256, 0, ss>>>(rp);
                else
                    rad_gemm2_kernel<<<g2, RTHREADS, 0, ss>>>(rp);
            }
            prof_end(tk, ss);
            rec_event(ev_join, ss, capturing);
            count_launch(((no_scan_planes || planes_used) ? 1 : 0) + (which & 1) + ((which >> 1) & 1));
            return cuda_check(cudaGetLastError(), "radius");
        }
        fused_planes_kernel<<<blocks_for(M * K, 256), 256, 0, ss>>>(av, M, K, 1, ec1, ec2, da1, da2, nullptr, nullptr);
        fused_planes_kernel<<<blocks_for(K * N, 256), 256, 0, ss>>>(bv, K, N, 0, fc1, fc2, db1, db2, nullptr, nullptr);
        // sparse products first, as 128-thread blocks small enough (registers, ~29 KB
        // smem) to share an SM with a band-GEMM CTA; the dense variants (which stand
        // down unless the device picked them) last
        static const bool carve = [] {
            cudaFuncSetAttribute(rad_spcol_v3_kernel<2, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            cudaFuncSetAttribute(rad_sprow_v3_kernel<2, 128>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
            return true;
        }();
        (void)carve;
        const int tk1 = prof_begin("rad_gemm", ss);
        rad_spcol_v3_kernel<2, 128><<<(unsigned)N, 128, 0, ss>>>(da1, db1, M, N, K, ec1, fc1, r1b, r1f, mw1);
        rad_sprow_v3_kernel<2, 128><<<(unsigned)M, 128, 0, ss>>>(da2, db2, M, N, K, ec2, fc2, r2b, r2f, mw2);
        rad_gemm_kernel<<<dim3(blocks_for(N, RT), blocks_for(M, RT)), RTHREADS, 0, ss>>>(da1, db1, M, N, K, ec1, fc1,
                                                                                       r1b, r1f, 0, 1, mw1);
        rad_gemm_kernel<<<dim3(blocks_for(N, RT), blocks_for(M, RT)), RTHREADS, 0, ss>>>(da2, db2, M, N, K, ec2, fc2,
                                                                                       r2b, r2f, 0, 0, mw2);
        prof_end(tk1, ss);
        prof_end(tk, ss);
        rec_event(ev_join, ss, capturing);
        count_launch(6);
        return cuda_check(cudaGetLastError(), "radius");
    };

    // graph cache lookup (profiling records per-launch events: eager then)
    const bool use_graphs = !no_graphs && !prof_enabled() && spec && sncw;
    std::vector<int64_t> key;
    if (use_graphs) {
        const apb_balls* bs[3] = {&A->b, &B->b, &C->b};
        key = {M, K, N, prec, sncw, (int64_t)scratch().gen, planes_used ? 1 : 0};
        for (const apb_balls* x : bs)
            key.insert(key.end(), {(int64_t)x->mant, (int64_t)x->exp, (int64_t)x->kind, (int64_t)x->rad_man,
                                   (int64_t)x->rad_exp, (int64_t)x->L});
    }
    GraphSet* gs = nullptr;
    if (use_graphs) {
        auto it = graphs().sets.find(key);
        if (it != graphs().sets.end() && it->second.g1 && it->second.gr) gs = &it->second;
    }
    int rc;
    cudaStream_t side = side_stream();
    static const bool no_spec_step = std::getenv("APB_NO_SPEC_STEP") != nullptr;  // test hook
    const auto g1s_it = gs ? gs->g1s.find(gs->k2s) : std::map<std::vector<int64_t>, std::pair<cudaGraphExec_t, int64_t>>::iterator{};
    const bool full_spec = gs && g1s_it != gs->g1s.end() && !no_spec_step;
    const std::vector<int64_t> k2_spec = full_spec ? gs->k2s : std::vector<int64_t>{};
    if (full_spec) {
        if (cudaGraphLaunch(g1s_it->second.first, st) != cudaSuccess) return cuda_check(cudaGetLastError(), "graph G1S");
        launch_count_adjust(g1s_it->second.second);
    } else if (gs) {
        if (cudaGraphLaunch(gs->g1, st) != cudaSuccess) return cuda_check(cudaGetLastError(), "graph G1");
        cudaStreamWaitEvent(side, ev_fin, 0);
        if (cudaGraphLaunch(gs->gr, side) != cudaSuccess) return cuda_check(cudaGetLastError(), "graph GR");
        launch_count_adjust(gs->n1 + gs->nr);
    } else {
        if ((rc = phase1(st, false))) return rc;
        if (spec) {
            cudaStreamWaitEvent(side, ev_fin, 0);
            if ((rc = phaseR(side, false))) return rc;
        }
        if (use_graphs) {  // capture for the next call with these operands
            if (graphs().sets.size() > 64) graphs().clear();
            GraphSet& ng = graphs().sets[key];
            ng.g1 = capture([&](cudaStream_t cs) { return phase1(cs, true); }, &ng.n1);
            ng.gr = capture([&](cudaStream_t cs) { return phaseR(cs, true); }, &ng.nr);
            gs = &ng;
        }
    }
    htrace().mark("scan_launched");
    if ((rc = cuda_check(cudaEventSynchronize(ev_plan), "matmul plan"))) return rc;
    htrace().mark("synced");
    const ScanSummary hsum = *hs;
    long long hw1[4], hw2[4];
    for (int q = 0; q < 4; q++) {
        hw1[q] = hw[q];
        hw2[q] = hw[4 + q];
    }
    Plan P;
    if ((rc = plan_finish(A, B, prec, hsum, P, st))) return rc;
    htrace().mark("planned");
    if (P.special) {  // src/matmul.cpp:455-458
        if (spec) cudaStreamWaitEvent(st, ev_join, 0);  // the speculative radius still reads scratch
        return classical(A, B, prec, C, st);
    }
    stats().block_calls++;
    stats().last_block_count = P.steps.size() / 3;
    // R_C += |A| R_B + R_A (|B| + R_B): FP64 work (independent of the midpoint product)
    const bool rad_multi = hw1[0] > 900 || hw1[1] > 900 || hw2[0] > 900 || hw2[1] > 900;
    // the speculative radius used the scan's uncentred planes: void if an operand
    // exponent was too far out (redo with centred planes, like a multi-block radius)
    static const bool no_scan_planes_h = std::getenv("APB_NO_SCAN_PLANES") != nullptr;
    // which radius kernels the device picks for this call's operands (rad_variant on the host copy
    // of the counts): the fused step's graph holds only those, so it is keyed on them too, and a
    // replay whose graph lacks a kernel these operands need redoes the radius
    static const bool rad_both = std::getenv("APB_RAD_BOTH") != nullptr;  // test hook: always launch both
    const int rv1 = rad_variant(hw1, M, K, N, 1), rv2 = rad_variant(hw2, M, K, N, 0);
    const int rad_which = rad_both ? 3 : ((rv1 == 0 || rv2 == 1) ? 1 : 0) | ((rv1 == 2 || rv2 == 2) ? 2 : 0);
    const bool rad_missing = full_spec && k2_spec.size() > 2 && (rad_which & ~(int)k2_spec[2]) != 0;
    const bool rad_redo = rad_multi || (!no_scan_planes_h && !planes_used && hsum.rad_centred) || rad_missing;
    want_planes = hsum.rad_centred != 0 && !rad_multi;
    const bool single = P.steps.size() == 3 && P.steps[0] == 0 && P.steps[1] == A->cols && P.steps[2] == 0;
    // slice planes the speculative pack of this call wrote: the fused step's graph writes the
    // speculated counts (early pack), every other path all template planes
    const int planes_a = (full_spec && early_ok) ? (int)k2_spec[0] : 8 * sncw;
    const int planes_b = (full_spec && early_ok) ? (int)k2_spec[1] : 8 * sncw;
    const bool prepacked = single && sncw && slices_for(P.maxw_a) <= planes_a && slices_for(P.maxw_b) <= planes_b;
    static const bool no_fuse = std::getenv("APB_NO_RAD_FUSE") != nullptr;  // test hook
    auto phase2 = [&](cudaStream_t s, bool capturing) -> int {
        RadFuse fz{r1b, r1f, r2b, r2f, ev_join, capturing, false};
        int rc2 = scaled_block(A, B, 0, K, prec, C, true, P.maxw_a, P.maxw_b, RW.top[0], RW.bot[0], CW.top[0],
                               CW.bot[0], nullptr, 0, nullptr, nullptr, s, nullptr, true, no_fuse ? nullptr : &fz);
        if (rc2) return rc2;
        if (fz.used) return cuda_check(cudaGetLastError(), "block matmul");
        wait_event(s, ev_join, capturing);
        const int tk_comb = prof_begin("combine", s);
        rad_combine_kernel<<<blocks_for(M * N, 256), 256, 0, s>>>(out_of(&C->b), M * N, r1b, r1f, r2b, r2f);
        prof_end(tk_comb, s);
        count_launch();
        return cuda_check(cudaGetLastError(), "block matmul");
    };
    if (full_spec) {
        const std::vector<int64_t> k2 = {slices_for(P.maxw_a), slices_for(P.maxw_b), rad_which};
        gs->k2s = k2;
        if (!rad_redo && prepacked && k2 == k2_spec) {  // the whole step already ran in G1S
            stats().int_gemm_products++;
            stats().last_height_a = (uint64_t)P.maxw_a;
            stats().last_height_b = (uint64_t)P.maxw_b;
            stats().last_slices_a = (uint64_t)k2[0];
            stats().last_slices_b = (uint64_t)k2[1];
            htrace().mark("done");
            htrace().flush();
            return APB_OK;
        }
        // the GEMM / recombine of G1S stood down (or the plan is not single-block):
        // continue below exactly as after G1 + GR (whose work G1S contains)
    }
    if (gs && spec && !rad_redo && prepacked) {  // the speculation held: G2
        const std::vector<int64_t> k2 = {slices_for(P.maxw_a), slices_for(P.maxw_b), rad_which};
        auto it = gs->g2.find(k2);
        gs->k2s = k2;
        if (it != gs->g2.end() && !full_spec && !gs->g1s.count(k2) && !no_spec_step) {
            // capture the fused single-graph step for the next call with these operands
            static cudaEvent_t ev_rdone = make_event();
            int64_t ns = 0;
            const uint64_t gemm_products = stats().int_gemm_products;
            cudaGraphExec_t g1 = capture(
                [&](cudaStream_t cs) -> int {
                    // APB_RAD_MAIN=1: radius products in stream order between the scan and the
                    // pack (measured 1 us slower than the side branch below, which overlaps them
                    // with the pack's tail)
                    static const bool rad_main = std::getenv("APB_RAD_MAIN") != nullptr;
                    if (rad_main && !std::getenv("APB_RAD_BESIDE")) {
                        const std::function<int(cudaStream_t)> radmid = [&](cudaStream_t ms) {
                            const int q = phaseR(ms, true);
                            cudaEventRecord(ev_rdone, ms);
                            return q;
                        };
                        int r = phase1(cs, true, &radmid);
                        if (r) return r;
                        RadFuse fz{r1b, r1f, r2b, r2f, ev_rdone, false, false};
                        r = scaled_block(A, B, 0, K, prec, C, true, P.maxw_a, P.maxw_b, RW.top[0], RW.bot[0],
                                         CW.top[0], CW.bot[0], nullptr, 0, nullptr, nullptr, cs, nullptr, true, &fz,
                                         &sum->maxw_a);
                        if (!r && !fz.used) {  // recombine16 did not fold the radius: combine here
                            rad_combine_kernel<<<blocks_for(M * N, 256), 256, 0, cs>>>(out_of(&C->b), M * N, r1b,
                                                                                        r1f, r2b, r2f);
                            count_launch();
                        }
                        return r;
                    }
                    int r = phase1(cs, true, nullptr, (int)k2[0], (int)k2[1]);  // (k2: this call's slice counts)
                    if (r) return r;
                    // radius branch: planes beside the pack, products before the GEMM, which
                    // waits for them (measured fastest: squeezed beside a GEMM CTA, one block
                    // per SM, the products outlast the GEMM).  APB_RAD_BESIDE=1: products
                    // issued after the pack, next to the GEMM (with APB_BAND_MAXNREG=144 builds)
                    static const bool rad_first = std::getenv("APB_RAD_BESIDE") == nullptr;
                    static cudaEvent_t ev_packed = make_event();
                    cudaStreamWaitEvent(side, ev_fork, 0);  // the planes beside the pack
                    if (!rad_first) cudaEventRecord(ev_packed, cs);
                    // APB_RAD_QUAD=1 APB_RAD_QUAD_BESIDE=1: the sparse radius products leave the side
                    // branch (which keeps the list compaction and the dense variants) and run beside
                    // the GEMM, launched right behind it on its stream as a programmatic dependent.
                    // Measured at config 3: the GEMM starts 20 us earlier but a GEMM CTA sharing its
                    // SM slows from 92 to 107 us whatever the co-resident warps execute (shuffles and
                    // shared loads go through the datapath the MMA operand fetch keeps ~75% busy),
                    // net 193 -> 191 us; not the default
                    static const bool beside = std::getenv("APB_RAD_QUAD_BESIDE") != nullptr && rad_first;
                    RadDefer dfr;
                    if ((r = phaseR(side, true, rad_first ? nullptr : ev_packed, beside ? &dfr : nullptr, rad_which))) return r;
                    cudaEventRecord(ev_rdone, side);
                    // small dense radius products (rad_gemm2s: config 2) fit beside the GEMM's CTAs
                    // and take longer than the GEMM: the GEMM does not wait for them, the recombine does
                    static const bool no_rad_along = std::getenv("APB_NO_RAD_ALONG") != nullptr;  // test hook
                    const dim3 rg2(blocks_for(N, RT), blocks_for(M, RT), 2);
                    const bool rad_along = !no_rad_along && rad_which == 2 && !std::getenv("APB_RAD_NO_SMALL") &&
                                           (int64_t)rg2.x * rg2.y * 2 < RAD_SMALL_TILES && !planes_used;
                    const bool join_first = rad_first && !rad_along;
                    if (join_first) cudaStreamWaitEvent(cs, ev_rdone, 0);
                    RadFuse fz{r1b, r1f, r2b, r2f, ev_rdone, false, false};
                    fz.joined = join_first;  // (the wait above; keeps the recombine right behind the GEMM)
                    const std::function<int()> rad_hook = [&]() -> int { return rad_quad_launch(dfr.rp, dfr.rl, cs, true); };
                    r = scaled_block(A, B, 0, K, prec, C, true, P.maxw_a, P.maxw_b, RW.top[0], RW.bot[0],
                                     CW.top[0], CW.bot[0], nullptr, 0, nullptr, nullptr, cs,
                                     dfr.ready ? &rad_hook : nullptr, true, &fz, &sum->maxw_a);
                    if (!r && !fz.used) r = APB_ERR_UNSUPPORTED;  // needs the fused recombine
                    cudaStreamWaitEvent(cs, ev_rdone, 0);           // rejoin the radius branch
                    return r;
                },
                &ns);
            stats().int_gemm_products = gemm_products;
            if (g1) gs->g1s[k2] = {g1, ns};
        }
        if (it != gs->g2.end() && !full_spec) {
            // host-side effects of scaled_block that a replay skips
            stats().int_gemm_products++;
            stats().last_height_a = (uint64_t)P.maxw_a;
            stats().last_height_b = (uint64_t)P.maxw_b;
            stats().last_slices_a = (uint64_t)slices_for(P.maxw_a);
            stats().last_slices_b = (uint64_t)slices_for(P.maxw_b);
            if (cudaGraphLaunch(it->second.first, st) != cudaSuccess) return cuda_check(cudaGetLastError(), "graph G2");
            launch_count_adjust(it->second.second);
            htrace().mark("done");
            htrace().flush();
            return APB_OK;
        }
        if ((rc = phase2(st, false))) return rc;
        if (it == gs->g2.end()) {
            int64_t n2 = 0;
            const uint64_t gemm_products = stats().int_gemm_products;
            cudaGraphExec_t g2 = capture([&](cudaStream_t cs) { return phase2(cs, true); }, &n2);
            stats().int_gemm_products = gemm_products;  // the capture pass ran no product
            if (g2) gs->g2[k2] = {g2, n2};
        }
        htrace().mark("done");
        htrace().flush();
        return APB_OK;
    }
    if (spec && rad_redo) cudaStreamWaitEvent(st, ev_join, 0);  // speculation void: redo below
    const int order = rad_redo ? 1 : rad_order;
    cudaStream_t rs = (order == 1 || order == 3) ? st : side;  // multi-block radius syncs its stream
    bool rad_done = spec && !rad_redo;
    std::function<int()> launch_radius = [&]() -> int {
        if (rad_done) return APB_OK;
        rad_done = true;
        int rc2;
        const int tk_rad = prof_begin("radius", rs);
        if (!rad_multi) {  // exact double planes of both radius products
            fused_planes_kernel<<<blocks_for(M * K, 256), 256, 0, rs>>>(av, M, K, 1, ec1, ec2, da1, da2, nullptr, nullptr);
            fused_planes_kernel<<<blocks_for(K * N, 256), 256, 0, rs>>>(bv, K, N, 0, fc1, fc2, db1, db2, nullptr, nullptr);
            count_launch(2);
        }
        if ((rc2 = radius_compute(A, B, 0, 2, 0, hw1, r1b, r1f, rs, 1))) return rc2;  // |A| plane transposed
        if ((rc2 = radius_compute(A, B, 1, 3, 1, hw2, r2b, r2f, rs))) return rc2;
        prof_end(tk_rad, rs);
        if (rs != st) cudaEventRecord(ev_join, rs);
        return APB_OK;
    };
    if ((order == 0 || order == 3) && (rc = launch_radius())) return rc;
    const std::function<int()>* hook = order == 2 ? &launch_radius : nullptr;
    bool first = true;
    for (size_t s = 0; s < P.steps.size(); s += 3) {
        const int64_t lo = P.steps[s], hi = P.steps[s + 1];
        if (P.steps[s + 2]) {
            if (first) {  // C starts as exact zeros
                cudaMemsetAsync(C->b.kind, 0, (size_t)M * N, st);
                cudaMemsetAsync(C->b.rad_man, 0, (size_t)M * N * 4, st);
                cudaMemsetAsync(C->b.exp, 0, (size_t)M * N * 8, st);
                cudaMemsetAsync(C->b.rad_exp, 0, (size_t)M * N * 8, st);
                cudaMemsetAsync(C->b.mant, 0, (size_t)M * N * 8 * C->b.L, st);
            }
            if ((rc = basecase(A, B, lo, hi, prec, C, st))) return rc;
        } else {
            if (single) {
                rc = scaled_block(A, B, lo, hi, prec, C, first, P.maxw_a, P.maxw_b, RW.top[0], RW.bot[0],
                                  CW.top[0], CW.bot[0], nullptr, 0, nullptr, nullptr, st, hook, prepacked);
            } else {
                rc = scaled_block(A, B, lo, hi, prec, C, first, 0, 0, nullptr, nullptr, nullptr, nullptr,
                                  nullptr, 0, nullptr, nullptr, st);
            }
            if (rc) return rc;
        }
        first = false;
    }
    if ((rc = launch_radius())) return rc;  // order 1 (or no GEMM ran)
    if (rs != st) cudaStreamWaitEvent(st, ev_join, 0);
    const int tk_comb = prof_begin("combine", st);
    rad_combine_kernel<<<blocks_for(M * N, 256), 256, 0, st>>>(out_of(&C->b), M * N, r1b, r1f, r2b, r2f);
    prof_end(tk_comb, st);
    count_launch();
    htrace().mark("done");
    htrace().flush();
    return cuda_check(cudaGetLastError(), "block matmul");
}

}  // namespace

int matmul_launch(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
                  cudaStream_t st) {
    if (A->rows * B->cols == 0) return APB_OK;
    if (A->cols == 0 || algo == APB_MM_CLASSICAL) return classical(A, B, prec, C, st);
    if (algo == APB_MM_AUTO) {  // matmul_dispatch_cutoff (src/matmul.cpp:517-531)
        int64_t cut = prec <= 64 ? 60 : prec <= 128 ? 56 : prec <= 256 ? 52 : prec <= 512 ? 48 : prec <= 1024 ? 44 : 40;
        int64_t mind = std::min(A->rows, std::min(A->cols, B->cols));
        if (mind <= cut) return classical(A, B, prec, C, st);
    }
    return block_matmul(A, B, prec, C, st);
}

}  // namespace apb

using namespace apb;

extern "C" {

int apb_matmul_complex(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre, const apb_mat* Bim,
                       int64_t prec, int algo, apb_mat* Cre, apb_mat* Cim, void* stream) {
    ApiLock api_lock;
    cudaStream_t st = (cudaStream_t)stream;
    if (!Are || !Aim || !Bre || !Bim || !Cre || !Cim || Are->cols != Bre->rows || Aim->cols != Bim->rows ||
        Are->rows != Aim->rows || Bre->cols != Bim->cols) {
        set_error("matmul: dimension mismatch");
        return APB_ERR_INVALID;
    }
    if (prec < 2) prec = 2;
    const int64_t M = Are->rows, N = Bre->cols;
    const int L = (int)((prec + 63) / 64);
    // four real products, each rounded to prec (src/matmul.cpp:538-541)
    static std::vector<void*> bufs(20, nullptr);
    static std::vector<size_t> caps(20, 0);
    auto get = [&](int k, size_t bytes) -> void* {
        if (caps[k] < bytes) {
            if (bufs[k]) {
                cudaStreamSynchronize(st);
                cudaFree(bufs[k]);
            }
            if (cudaMalloc(&bufs[k], bytes) != cudaSuccess) return nullptr;
            caps[k] = bytes;
        }
        return bufs[k];
    };
    apb_mat P4[4];
    for (int q = 0; q < 4; q++) {
        apb_balls& b = P4[q].b;
        b.count = M * N;
        b.L = L;
        b.mant = (uint64_t*)get(5 * q, (size_t)M * N * L * 8);
        b.exp = (int64_t*)get(5 * q + 1, (size_t)M * N * 8);
        b.kind = (uint8_t*)get(5 * q + 2, (size_t)M * N);
        b.rad_man = (uint32_t*)get(5 * q + 3, (size_t)M * N * 4);
        b.rad_exp = (int64_t*)get(5 * q + 4, (size_t)M * N * 8);
        if (!b.mant || !b.exp || !b.kind || !b.rad_man || !b.rad_exp) {
            set_error("out of device memory");
            return APB_ERR_CUDA;
        }
        P4[q].rows = M;
        P4[q].cols = N;
    }
    const apb_mat* lhs[4] = {Are, Aim, Are, Aim};
    const apb_mat* rhs[4] = {Bre, Bim, Bim, Bre};  // AC, BD, AD, BC
    for (int q = 0; q < 4; q++) {
        int rc = matmul_launch(lhs[q], rhs[q], prec, algo, &P4[q], st);
        if (rc) return rc;
    }
    int* status = workspace().status_dev;
    ball_addsub_kernel<<<blocks_for(M * N, 128), 128, 0, st>>>(view_of(&P4[0].b), view_of(&P4[1].b), 1, M * N,
                                                               prec, out_of(&Cre->b), status);
    ball_addsub_kernel<<<blocks_for(M * N, 128), 128, 0, st>>>(view_of(&P4[2].b), view_of(&P4[3].b), 0, M * N,
                                                               prec, out_of(&Cim->b), status);
    count_launch(2);
    return cuda_check(cudaGetLastError(), "complex matmul");
}

// IMAD-limb baseline of apb_block_int_product: same scan, 32-bit limb planes,
// CUDA-core product (imad_gemm_kernel); the GEMM time goes to *gemm_ms if given
int imad_block_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi, int64_t* row_scale,
                       int64_t* col_scale, uint64_t* out, int64_t out_limbs, float* gemm_ms, cudaStream_t st) {
    const int64_t M = A->rows, N = B->cols, w = hi - lo;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int64_t* rt = sbuf<int64_t>(S_RTOP, M, st);
    int64_t* rb = sbuf<int64_t>(S_RBOT, M, st);
    int64_t* ct = sbuf<int64_t>(S_CTOP, N, st);
    int64_t* cb = sbuf<int64_t>(S_CBOT, N, st);
    ScanSummary* sum = sbuf<ScanSummary>(S_SUM, 1, st);
    if (!rt || !rb || !ct || !cb || !sum) return APB_ERR_CUDA;
    cudaMemsetAsync(sum, 0, sizeof(ScanSummary), st);
    scan_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, A->cols, lo, hi, rt, rb, sum);
    scan_cols(b, A->cols, N, lo, hi, ct, cb, sum, st);
    ScanSummary h;
    cudaMemcpyAsync(&h, sum, sizeof h, cudaMemcpyDeviceToHost, st);
    int rc = cuda_check(cudaStreamSynchronize(st), "imad scan");
    if (rc) return rc;
    const int Qn = (int)((std::max(h.maxw_a, h.maxw_b) + 31) / 32);
    int Q = 0;
    for (int c : {4, 6, 8, 11, 14, 19})
        if (!Q && Qn <= c) Q = c;
    if (!Q) {
        set_error("imad baseline: entry height above 19 limbs");
        return APB_ERR_UNSUPPORTED;
    }
    uint32_t* Al = sbuf<uint32_t>(S_APACK, (size_t)Q * M * w, st);
    uint32_t* Bl = sbuf<uint32_t>(S_BPACK, (size_t)Q * w * N, st);
    uint8_t* As = sbuf<uint8_t>(S_TW, (size_t)M * w, st);
    uint8_t* Bs = sbuf<uint8_t>(S_TC, (size_t)w * N, st);
    if (!Al || !Bl || !As || !Bs) return APB_ERR_CUDA;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const dim3 g((unsigned)((N + 15) / 16), (unsigned)((M + 15) / 16));
    const dim3 g2((unsigned)((N + 31) / 32), (unsigned)((M + 31) / 32));
    const dim3 g21((unsigned)((N + 15) / 16), (unsigned)((M + 31) / 32));
#define APB_IMAD_Q(QQ)                                                                                       \
    case QQ:                                                                                                 \
        limb_pack_kernel<QQ><<<blocks_for(M * w, 256), 256, 0, st>>>(a, M, w, A->cols, lo, 1, rt, rb, Al, As,  \
                                                                       row_scale);                            \
        limb_pack_kernel<QQ><<<blocks_for(w * N, 256), 256, 0, st>>>(b, w, N, N, lo, 0, ct, cb, Bl, Bs,        \
                                                                       col_scale);                            \
        cudaEventRecord(e0, st);                                                                              \
        if constexpr (QQ <= 6)                                                                                \
            imad_gemm_kernel<QQ, 2, 2><<<g2, 256, 0, st>>>(Al, As, Bl, Bs, M, N, w, out, (int)out_limbs);        \
        else if constexpr (QQ <= 8)                                                                           \
            imad_gemm_kernel<QQ, 2, 1><<<g21, 256, 0, st>>>(Al, As, Bl, Bs, M, N, w, out, (int)out_limbs);       \
        else                                                                                                  \
            imad_gemm_kernel<QQ, 1, 1><<<g, 256, 0, st>>>(Al, As, Bl, Bs, M, N, w, out, (int)out_limbs);         \
        cudaEventRecord(e1, st);                                                                              \
        break;
    switch (Q) {
        APB_IMAD_Q(4)
        APB_IMAD_Q(6)
        APB_IMAD_Q(8)
        APB_IMAD_Q(11)
        APB_IMAD_Q(14)
        APB_IMAD_Q(19)
    }
#undef APB_IMAD_Q
    count_launch(3);
    rc = cuda_check(cudaEventSynchronize(e1), "imad gemm");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (gemm_ms) *gemm_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return rc;
}

int apb_block_int_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi, int64_t* row_scale,
                          int64_t* col_scale, uint64_t* out, int64_t out_limbs, void* stream) {
    ApiLock api_lock;
    if (!A || !B || A->cols != B->rows || lo < 0 || hi > A->cols || hi <= lo) {
        set_error("int_matmul: dimension mismatch");
        return APB_ERR_INVALID;
    }
    return scaled_block(A, B, lo, hi, 0, nullptr, true, 0, 0, nullptr, nullptr, nullptr, nullptr,
                        (int64_t*)out, (int)out_limbs, row_scale, col_scale, (cudaStream_t)stream);
}

int apb_block_int_product_imad(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi, int64_t* row_scale,
                               int64_t* col_scale, uint64_t* out, int64_t out_limbs, float* gemm_ms, void* stream) {
    ApiLock api_lock;
    if (!A || !B || A->cols != B->rows || lo < 0 || hi > A->cols || hi <= lo) {
        set_error("int_matmul: dimension mismatch");
        return APB_ERR_INVALID;
    }
    return imad_block_product(A, B, lo, hi, row_scale, col_scale, out, out_limbs, gemm_ms, (cudaStream_t)stream);
}

int apb_plan_blocks(const apb_mat* A, const apb_mat* B, int64_t prec, int64_t* steps_out, int64_t max_steps,
                    int64_t* n_steps, void* stream) {
    ApiLock api_lock;
    if (!A || !B || A->cols != B->rows) {
        set_error("plan_blocks: dimension mismatch");
        return APB_ERR_INVALID;
    }
    Plan P;
    int rc = plan(A, B, prec, P, (cudaStream_t)stream);
    if (rc) return rc;
    *n_steps = (int64_t)P.steps.size() / 3;
    for (int64_t i = 0; i < *n_steps && i < max_steps; i++)
        for (int q = 0; q < 3; q++) steps_out[3 * i + q] = P.steps[3 * i + q];
    return APB_OK;
}

int apb_matmul_plan_info(const apb_mat* A, const apb_mat* B, int64_t prec, apb_plan_info* out,
                         void* stream) {
    ApiLock api_lock;
    if (!A || !B || !out || A->cols != B->rows) {
        set_error("plan_info: dimension mismatch");
        return APB_ERR_INVALID;
    }
    cudaStream_t st = (cudaStream_t)stream;
    std::memset(out, 0, sizeof *out);
    Plan P;
    int rc = plan(A, B, prec, P, st);
    if (rc) return rc;
    out->special = P.special ? 1 : 0;
    out->n_blocks = (int64_t)P.steps.size() / 3;
    out->entry_prec_a = P.prec_a;
    out->entry_prec_b = P.prec_b;
    out->max_width_a = P.maxw_a;
    out->max_width_b = P.maxw_b;
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    BallsView a = view_of(&A->b), b = view_of(&B->b);
    int64_t* ecen = sbuf<int64_t>(S_CEN_E, M, st);
    int64_t* fcen = sbuf<int64_t>(S_CEN_F, N, st);
    long long* mw = sbuf<long long>(S_SUM, 4, st);
    cudaMemsetAsync(mw, 0, 4 * sizeof(long long), st);
    rad_center_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, 0, K, 0, ecen, mw);
    rad_center_rows_kernel<<<blocks_for(M, 8), 256, 0, st>>>(a, M, K, 0, K, 1, ecen, mw + 1);
    rad_center_cols(b, K, N, 0, K, 2, fcen, mw + 2, st);
    rad_center_cols(b, K, N, 0, K, 3, fcen, mw + 3, st);
    count_launch(2);
    long long hw[4];
    cudaMemcpyAsync(hw, mw, sizeof hw, cudaMemcpyDeviceToHost, st);
    if ((rc = cuda_check(cudaStreamSynchronize(st), "plan info"))) return rc;
    out->radius_single = (hw[0] <= 900 && hw[1] <= 900 && hw[2] <= 900 && hw[3] <= 900) ? 1 : 0;
    return APB_OK;
}

int apb_radius_matmul_upper(const uint32_t* p_man, const int64_t* p_exp, const uint32_t* q_man,
                            const int64_t* q_exp, int64_t m, int64_t n, int64_t k, uint32_t* out_man,
                            int64_t* out_exp, void* stream) {
    ApiLock api_lock;
    // P and Q are carried as the radius planes of ball matrices whose
    // midpoints are never read (operand kinds 1 and 2 of rad_operand)
    if (!p_man || !p_exp || !q_man || !q_exp || !out_man || !out_exp || m < 0 || n < 0 || k < 0) {
        set_error("radius_matmul_upper: invalid arguments");
        return APB_ERR_INVALID;
    }
    apb_mat P{}, Q{};
    static uint64_t dummy_mant;
    P.b.mant = Q.b.mant = &dummy_mant;
    P.b.exp = Q.b.exp = (int64_t*)p_exp;
    P.b.kind = Q.b.kind = (uint8_t*)p_man;
    P.b.L = Q.b.L = 1;
    P.b.rad_man = (uint32_t*)p_man;
    P.b.rad_exp = (int64_t*)p_exp;
    Q.b.rad_man = (uint32_t*)q_man;
    Q.b.rad_exp = (int64_t*)q_exp;
    P.rows = m;
    P.cols = n;
    Q.rows = n;
    Q.cols = k;
    if (m * k == 0) return APB_OK;
    if (n == 0) {
        cudaMemsetAsync(out_man, 0, (size_t)m * k * 4, (cudaStream_t)stream);
        cudaMemsetAsync(out_exp, 0, (size_t)m * k * 8, (cudaStream_t)stream);
        return APB_OK;
    }
    return radius_product(&P, &Q, 1, 2, out_man, out_exp, (cudaStream_t)stream);
}

}  // extern "C"
