// dot_kernels.cu - batched fused ball dot products (K1/K2) for sm_100a.
//
// Restates Algorithm 1 of the reference (src/dot.cpp, paths relative to
// /root/reference/proj) for a batch of independent dots:
//
//   dot_small<L,NS,TPL>  one warp per dot, lanes stride over the terms.
//       Pass 1 (setup_core, src/dot.cpp:72-134) is a warp reduction of
//       e_max / e_min / e_rad / n_nonzero / fallback; every lane then derives
//       the identical plan (p_eff, n_s, e_s).  Pass 2 computes each lane's
//       terms into a private NS-limb two's complement accumulator held in
//       registers (dot_accumulate_term + accumulate_aligned, src/dot.cpp:
//       139-273), plus the integer ulp count `err` and the scaled radius sum
//       `srad` (src/dot.cpp:282-295, 346-358).  The lane accumulators are
//       combined by a warp-shuffle carry-propagating reduction (two's
//       complement addition mod 2^(64 n_s) is associative, so the result is
//       bit-identical to the reference's sequential order).  Lane 0 runs
//       dot_finalize (src/dot.cpp:306-321).
//       Per-term contribution: with the operands in L-limb top-aligned slots,
//       the (truncated) product P = A*B (2L limbs) enters the accumulator as
//       floor(P / 2^r), r = shift + 128 L - 64 n_s, and err += 1 iff the floor
//       dropped nonzero bits -- exactly the limb placement/drop rule of
//       accumulate_aligned.  The short product (mulhigh) never triggers here
//       (it needs n_s >= 25, src/dot.cpp:259).
//
//   dot_generic  one thread per dot, runtime limb counts in local memory: the
//       wide-precision path (any L, n_s, mulhigh_approx) and the special-value
//       fallback (ball_fallback_addmul, src/ball.cpp:21-36; src/dot.cpp:325-344).
//       In `fallback_only` mode it processes only dots the small kernel
//       flagged as Fallback.
//
//   dot_complex_generic  complex dots (src/dot.cpp:470-568): two accumulators
//       (re, im) over the 2N-term part views, thread per dot.

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <cstdlib>
#include <cuda_runtime.h>

#include "apb.h"
#include "apb_common.cuh"
#include "apb_internal.h"

namespace apb {

constexpr int64_t kExpCap = int64_t(1) << 60;  // src/dot.cpp:13
APB_DEV bool exp_huge(int64_t e) { return e > kExpCap || e < -kExpCap; }

struct DotArgs {
    BallsView x, y, init;
    bool has_init;
    BallsOut out;
    apb_dot_index idx;
    int64_t n, batch, prec;
    int mode;  // APB_DOT_BALL / APB_DOT_APPROX
    int subtract;
    int disable_reduction;
    apb_dot_state* state;
    uint64_t* acc;
    int64_t acc_stride;
    uint8_t* fb_flag;  // per dot: 1 = needs the fallback path
    int* status;
    // poly_mullow_classical mode (palen > 0): dot k runs over a[i0..i1] and
    // b[k-i0] downwards (src/poly.cpp:11-26), its length varies with k
    int64_t palen = 0, pblen = 0;
    int dpw = 32;  // dots per warp in dot_small_kernel (fewer for small batches)
    bool mant16 = false;  // x and y both 2-limb with 16-byte aligned mantissa arrays
};

// element index of term 0, the steps, and the term count of dot b
APB_DEV void dot_extent(const DotArgs& A, int64_t b, int64_t& ex0, int64_t& xs, int64_t& ey0, int64_t& ys,
                        int64_t& n) {
    if (A.palen > 0) {
        const int64_t i0 = b + 1 > A.pblen ? b + 1 - A.pblen : 0;
        const int64_t i1 = b < A.palen - 1 ? b : A.palen - 1;
        n = (i0 >= A.palen || i1 < i0) ? 0 : i1 - i0 + 1;
        ex0 = i0;
        xs = 1;
        ey0 = b - i0;
        ys = -1;
        return;
    }
    const int64_t bq = A.idx.bdiv == 1 ? b : b / A.idx.bdiv;
    const int64_t br = A.idx.bdiv == 1 ? 0 : b - bq * A.idx.bdiv;
    ex0 = A.idx.x_off + bq * A.idx.xs1 + br * A.idx.xs2;
    ey0 = A.idx.y_off + bq * A.idx.ys1 + br * A.idx.ys2;
    xs = A.idx.xstep;
    ys = A.idx.ystep;
    n = A.n;
}

APB_DEV int64_t x_elem(const apb_dot_index& ix, int64_t b, int64_t i) {
    return ix.x_off + (b / ix.bdiv) * ix.xs1 + (b % ix.bdiv) * ix.xs2 + i * ix.xstep;
}
APB_DEV int64_t y_elem(const apb_dot_index& ix, int64_t b, int64_t i) {
    return ix.y_off + (b / ix.bdiv) * ix.ys1 + (b % ix.bdiv) * ix.ys2 + i * ix.ystep;
}

// ---------------------------------------------------------------- plan

struct Plan {
    int64_t e_max, e_min, e_rad;
    uint64_t nnz;
    int64_t p_eff;
    int extend, padding;
    int n_s;
    int64_t e_s;
    int status;  // 0 proceed 1 fallback 2 zero
};

// tail of setup_core after the scan (src/dot.cpp:115-131)
APB_DEV Plan finish_plan(int64_t e_max, int64_t e_min, int64_t e_rad, uint64_t nnz, bool fb,
                         int64_t total, int64_t p, bool disable_reduction) {
    Plan pl;
    pl.e_max = e_max;
    pl.e_min = e_min;
    pl.e_rad = e_rad;
    pl.nnz = nnz;
    pl.p_eff = 2;
    pl.extend = pl.padding = 0;
    pl.n_s = 0;
    pl.e_s = 0;
    if (fb) {
        pl.status = 1;
        return pl;
    }
    if (e_max == INT64_MIN && e_rad == INT64_MIN) {
        pl.status = 2;
        return pl;
    }
    if (e_max == INT64_MIN) {
        p = 2;
    } else if (!disable_reduction) {
        if (e_rad != INT64_MIN && e_max - e_rad + 30 < p) p = e_max - e_rad + 30;
        if (e_min != INT64_MAX && e_max - e_min + 30 < p) p = e_max - e_min + 30;
        if (p < 2) p = 2;
    }
    pl.p_eff = p;
    pl.padding = 4 + (int)bitw64((uint64_t)total);
    pl.extend = (int)bitw64(nnz) + 1;
    int64_t ns = (p + pl.extend + pl.padding + 63) / 64;
    pl.n_s = (int)(ns < 2 ? 2 : ns);
    pl.e_s = e_max == INT64_MIN ? 0 : e_max + pl.extend;
    pl.status = 0;
    return pl;
}

APB_DEV void write_state(apb_dot_state* st, const Plan& pl, uint64_t err, uint64_t srad) {
    st->e_max = pl.e_max;
    st->e_min = pl.e_min;
    st->e_rad = pl.e_rad;
    st->n_nonzero = pl.nnz;
    st->p_eff = pl.p_eff;
    st->extend = pl.extend;
    st->padding = pl.padding;
    st->n_s = pl.n_s;
    st->e_s = pl.e_s;
    st->status = pl.status;
    st->_pad = 0;
    st->err = err;
    st->srad = srad;
}

// srad_add (src/dot.cpp:288-295); both factors are < 2^31 (one 32x32 multiply)
APB_DEV uint64_t srad_term(uint64_t ab, int64_t af, uint64_t bb, int64_t bf, int64_t e_rad) {
    int64_t d = e_rad - (af + bf);
    return d < 30 ? (((uint64_t)(uint32_t)ab * (uint32_t)bb) >> (30 + d)) + 1 : 1;
}

// dot_finalize (src/dot.cpp:306-321) given the reduced accumulator
template <int CAP>
__device__ void finalize_store(const Plan& pl, const uint64_t* s_in, uint64_t err, uint64_t srad,
                               int64_t p, bool with_radius, const BallsOut& out, int64_t b,
                               int* status) {
    if (p > pl.p_eff) p = pl.p_eff;
    if (p < 2) p = 2;
    uint64_t s[CAP];
    for (int i = 0; i < pl.n_s; i++) s[i] = s_in[i];
    int sign = 0;
    if (s[pl.n_s - 1] >> 63) {  // neg_in_place (include/apball/limb.hpp:180-187)
        int i = 0;
        while (i < pl.n_s && s[i] == 0) i++;
        if (i < pl.n_s) {
            s[i] = ~s[i] + 1;
            for (i++; i < pl.n_s; i++) s[i] = ~s[i];
        }
        sign = 1;
    }
    GFloat<CAP> mid;
    gf_normalize(mid, sign, pl.e_s, s, pl.n_s, status);
    Mag r = gf_round(mid, p, status);
    if (with_radius) {
        if (err) r = mag_add(r, mag_from_u64(err, pl.e_s - 64 * (int64_t)pl.n_s));
        if (srad) r = mag_add(r, mag_from_u64(srad, pl.e_rad - 30));
    } else {
        r = mag_zero();
    }
    gf_store(out, b, mid, r, status);
}

// ----------------------------------------------------------- term loads

template <int L>
struct Term {
    uint64_t xm[L], ym[L];
    int64_t ex, ey;
    uint8_t kx, ky;
    uint32_t rx, ry;
    int64_t fx, fy;
    bool neg;  // subtract flag of this term
};

template <int L>
APB_DEV void load_mant(uint64_t (&m)[L], const BallsView& a, int64_t e) {
    const int off = L - a.L;  // a.L <= L, top-aligned
    const uint64_t* src = a.mant + e * (int64_t)a.L;
#pragma unroll
    for (int j = 0; j < L; j++) m[j] = (j >= off) ? __ldg(src + (j - off)) : 0ull;
}

// term i of dot b from precomputed element indices (ex, ey): the metadata always,
// the mantissas only when `mant` (pass 1 needs them only for e_min)
template <int L>
APB_DEV void load_term_at(Term<L>& t, const DotArgs& A, int64_t b, int64_t i, int64_t ex, int64_t ey, bool mant,
                          int64_t n) {
    if (i < n) {
        t.kx = __ldg(A.x.kind + ex);
        t.ky = __ldg(A.y.kind + ey);
        t.ex = __ldg(A.x.exp + ex);
        t.ey = __ldg(A.y.exp + ey);
        t.rx = __ldg(A.x.rad_man + ex);
        t.ry = __ldg(A.y.rad_man + ey);
        t.fx = __ldg(A.x.rad_exp + ex);
        t.fy = __ldg(A.y.rad_exp + ey);
        if (mant) {
            load_mant<L>(t.xm, A.x, ex);
            load_mant<L>(t.ym, A.y, ey);
        }
        t.neg = A.subtract != 0;
    } else {  // the initial value as term N with y = 1 (src/dot.cpp:29-43)
        t.kx = __ldg(A.init.kind + b);
        t.ex = __ldg(A.init.exp + b);
        t.rx = __ldg(A.init.rad_man + b);
        t.fx = __ldg(A.init.rad_exp + b);
        load_mant<L>(t.xm, A.init, b);
        t.ky = APB_FINITE;
        t.ey = 1;
        t.ry = 0;
        t.fy = 0;
#pragma unroll
        for (int j = 0; j < L; j++) t.ym[j] = (j == L - 1) ? (1ull << 63) : 0ull;
        t.neg = false;
    }
}

template <int L>
APB_DEV void load_term(Term<L>& t, const DotArgs& A, int64_t b, int64_t i) {
    if (i < A.n) {
        const int64_t bq = A.idx.bdiv == 1 ? b : b / A.idx.bdiv;
        const int64_t br = A.idx.bdiv == 1 ? 0 : b - bq * A.idx.bdiv;
        const int64_t ex = A.idx.x_off + bq * A.idx.xs1 + br * A.idx.xs2 + i * A.idx.xstep;
        const int64_t ey = A.idx.y_off + bq * A.idx.ys1 + br * A.idx.ys2 + i * A.idx.ystep;
        t.kx = __ldg(A.x.kind + ex);
        t.ky = __ldg(A.y.kind + ey);
        t.ex = __ldg(A.x.exp + ex);
        t.ey = __ldg(A.y.exp + ey);
        t.rx = __ldg(A.x.rad_man + ex);
        t.ry = __ldg(A.y.rad_man + ey);
        t.fx = __ldg(A.x.rad_exp + ex);
        t.fy = __ldg(A.y.rad_exp + ey);
        load_mant<L>(t.xm, A.x, ex);
        load_mant<L>(t.ym, A.y, ey);
        t.neg = A.subtract != 0;
    } else {  // the initial value as term N with y = 1 (src/dot.cpp:29-43)
        t.kx = __ldg(A.init.kind + b);
        t.ex = __ldg(A.init.exp + b);
        t.rx = __ldg(A.init.rad_man + b);
        t.fx = __ldg(A.init.rad_exp + b);
        load_mant<L>(t.xm, A.init, b);
        t.ky = APB_FINITE;
        t.ey = 1;
        t.ry = 0;
        t.fy = 0;
#pragma unroll
        for (int j = 0; j < L; j++) t.ym[j] = (j == L - 1) ? (1ull << 63) : 0ull;
        t.neg = false;
    }
}

// minimal limb count of a top-aligned L-slot mantissa
template <int L>
APB_DEV int limb_count(const uint64_t (&m)[L]) {
    int z = 0;
    bool seen = false;
#pragma unroll
    for (int j = 0; j < L; j++) {
        if (!seen && m[j] == 0) z++;
        else seen = true;
    }
    return L - z;
}

struct ScanAcc {
    int64_t e_max, e_min, e_rad;
    uint64_t nnz;
    bool fb;
};

template <int L>
APB_DEV void scan_term(ScanAcc& s, const Term<L>& t, bool track_min, bool with_radius) {
    const int kx = t.kx & APB_KIND_MASK, ky = t.ky & APB_KIND_MASK;
    const bool xz = kx == APB_ZERO, yz = ky == APB_ZERO;
    if ((kx != APB_ZERO && kx != APB_FINITE) || (ky != APB_ZERO && ky != APB_FINITE)) {
        s.fb = true;
        return;
    }
    if ((!xz && exp_huge(t.ex)) || (!yz && exp_huge(t.ey))) {
        s.fb = true;
        return;
    }
    if (!xz && !yz) {
        s.nnz++;
        int64_t ee = t.ex + t.ey;
        s.e_max = ee > s.e_max ? ee : s.e_max;
        if (track_min) {
            int64_t lo = ee - 64 * (int64_t)(limb_count<L>(t.xm) + limb_count<L>(t.ym));
            s.e_min = lo < s.e_min ? lo : s.e_min;
        }
    }
    if (with_radius) {
        const bool rxz = t.rx == 0, ryz = t.ry == 0;
        if (t.rx == APB_RAD_INF || t.ry == APB_RAD_INF || (!rxz && exp_huge(t.fx)) ||
            (!ryz && exp_huge(t.fy))) {
            s.fb = true;
            return;
        }
        if (!ryz && !xz && t.ex + t.fy > s.e_rad) s.e_rad = t.ex + t.fy;
        if (!rxz && !yz && t.ey + t.fx > s.e_rad) s.e_rad = t.ey + t.fx;
        if (!rxz && !ryz && t.fx + t.fy > s.e_rad) s.e_rad = t.fx + t.fy;
    }
}

// Mag canonicalization of a loaded radius (Mag::from_parts): the SoA stores
// canonical mantissas, so (b, f) is used as is.

// ------------------------------------------------------- small kernel

template <int L, int NS>
struct Acc {
    uint64_t s[NS];
    uint64_t err;
    uint64_t srad;
};

// accumulate one nonzero term (dot_accumulate_term, src/dot.cpp:229-273)
template <int L, int NS>
APB_DEV void acc_term(Acc<L, NS>& a, const Term<L>& t, const Plan& pl) {
    const bool negate = t.neg ^ ((t.kx & APB_SIGN) != 0) ^ ((t.ky & APB_SIGN) != 0);
    const int64_t shift64 = pl.e_s - (t.ex + t.ey);
    if (shift64 >= 64 * (int64_t)pl.n_s) {
        a.err++;
        return;
    }
    const int shift = (int)shift64;  // 0 <= shift < 64 n_s (e_s >= every term's exponent)
    // operand truncation to ncap limbs (src/dot.cpp:248-253)
    const int p_t = 64 * pl.n_s - shift;
    const int ncap = (p_t + 63) / 64 + 1;
    uint64_t xa[L], yb[L];
    bool trunc = false;
#pragma unroll
    for (int j = 0; j < L; j++) {
        const bool keep = (L - j) <= ncap;  // slot j is within the top ncap slots
        xa[j] = keep ? t.xm[j] : 0ull;
        yb[j] = keep ? t.ym[j] : 0ull;
        trunc |= (!keep) && (t.xm[j] | t.ym[j]);
    }
    if (trunc) a.err++;
    // P = xa * yb, 2L limbs
    uint64_t P[2 * L];
#pragma unroll
    for (int k = 0; k < 2 * L; k++) P[k] = 0;
#pragma unroll
    for (int i = 0; i < L; i++) {
        uint64_t cy = 0;
#pragma unroll
        for (int j = 0; j < L; j++) {
            uint64_t lo, hi;
            mul64(xa[i], yb[j], lo, hi);
            uint64_t s1 = P[i + j] + lo;
            uint64_t c1 = s1 < lo;
            uint64_t s2 = s1 + cy;
            uint64_t c2 = s2 < cy;
            P[i + j] = s2;
            cy = hi + c1 + c2;  // cannot overflow: hi <= 2^64-2
        }
        P[i + L] = cy;
    }
    // contribution floor(P / 2^r), r = shift + 128 L - 64 n_s (>= 0 here: n_s <= 2L + 1
    // whenever the term is not dropped); word shift by a barrel of static selects
    const int r = shift + 128 * L - 64 * pl.n_s;
    if (r < 0) {  // window wider than the product: exact, shifted left
        const int rl = (-r) >> 6, rb = (-r) & 63;
        uint64_t Cl[NS];
#pragma unroll
        for (int j = 0; j < NS; j++) {
            uint64_t lo = 0, hi = 0;  // Cl[j] = bits of P << (-r) at word j
#pragma unroll
            for (int k = 0; k < 2 * L; k++) {
                if (k == j - rl) hi = P[k];
                if (k == j - rl - 1) lo = P[k];
            }
            Cl[j] = rb ? (hi << rb) | (lo >> (64 - rb)) : hi;
        }
        if (!negate)
            addn_mod<NS>(a.s, Cl);
        else
            subn_mod<NS>(a.s, Cl);
        return;
    }
    const int rl = r >> 6;
    const unsigned rb = (unsigned)(r & 63);
    // barrel: Q = P >> (64 rl) with sticky = OR of the dropped words
    constexpr int W = 2 * L;
    uint64_t Q[W];
    uint64_t sticky = 0;
#pragma unroll
    for (int k = 0; k < W; k++) Q[k] = P[k];
#pragma unroll
    for (int bit = 1; bit <= W - 1; bit <<= 1) {  // rl <= W - 1
        const bool on = (rl & bit) != 0;
        uint64_t drop = 0;
#pragma unroll
        for (int k = 0; k < W; k++)
            if (k < bit) drop |= Q[k];
        if (on) sticky |= drop;
#pragma unroll
        for (int k = 0; k < W; k++) {
            const uint64_t nv = (k + bit < W) ? Q[k + bit] : 0ull;
            Q[k] = on ? nv : Q[k];
        }
    }
    const bool inexact = sticky != 0 || (rb && (Q[0] & ((1ull << rb) - 1)) != 0);
    if (inexact) a.err++;
    uint64_t Cl[NS];
#pragma unroll
    for (int j = 0; j < NS; j++) {
        const uint64_t lo = j < W ? Q[j] : 0ull;
        const uint64_t hi = j + 1 < W ? Q[j + 1] : 0ull;
        Cl[j] = funnel_r(lo, hi, rb);
    }
    // two's complement add / subtract mod 2^(64 NS) (add_signed_range)
    if (!negate)
        addn_mod<NS>(a.s, Cl);
    else
        subn_mod<NS>(a.s, Cl);
}

// radius_pass_term (src/dot.cpp:346-358)
template <int L, int NS>
APB_DEV void rad_term(Acc<L, NS>& a, const Term<L>& t, const Plan& pl) {
    const bool xz = (t.kx & APB_KIND_MASK) == APB_ZERO, yz = (t.ky & APB_KIND_MASK) == APB_ZERO;
    if (t.ry != 0 && !xz) a.srad += srad_term((t.xm[L - 1] >> 34) + 1, t.ex, t.ry, t.fy, pl.e_rad);
    if (t.rx != 0 && !yz) a.srad += srad_term((t.ym[L - 1] >> 34) + 1, t.ey, t.rx, t.fx, pl.e_rad);
    if (t.rx != 0 && t.ry != 0) a.srad += srad_term(t.rx, t.fx, t.ry, t.fy, pl.e_rad);
}

APB_DEV int64_t warp_max(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
APB_DEV int64_t warp_min(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
APB_DEV uint64_t warp_sum(uint64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Per-warp batch of up to 32 dots: dot g's reduced accumulator is parked in
// lane g, and the 32 finalizes (normalize / truncate / Mag error terms) run
// in parallel at the end instead of serially on lane 0.
template <int L, int NS, int TPL>
__global__ void __launch_bounds__(128, (TPL > 0 ? 3 : 4)) dot_small_kernel(DotArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t b0 = warp_id * A.dpw;
    if (b0 >= A.batch) return;
    const int nd = (int)(A.batch - b0 < A.dpw ? A.batch - b0 : A.dpw);
    const bool with_radius = A.mode == APB_DOT_BALL;
    const bool track_min = A.prec > 128;

    // lane-parked results of dot b0 + lane
    Plan my_pl;
    uint64_t my_s[NS];
    uint64_t my_err = 0, my_srad = 0;
    my_pl.status = 2;

    for (int g = 0; g < nd; g++) {
        const int64_t b = b0 + g;
        // element indices of this lane's first term (index math once per dot)
        int64_t ex0, xst, ey0, yst, nb;
        dot_extent(A, b, ex0, xst, ey0, yst, nb);
        const int64_t total = nb + (A.has_init ? 1 : 0);
        ex0 += lane * xst;
        ey0 += lane * yst;
        const int64_t xstep32 = 32 * xst, ystep32 = 32 * yst;
        // ---- pass 1: setup scan
        ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
        Term<L> keep[TPL > 0 ? TPL : 1];
        if (TPL > 0) {
#pragma unroll
            for (int q = 0; q < (TPL > 0 ? TPL : 1); q++) {
                int64_t i = lane + 32 * (int64_t)q;
                if (i < total) {
                    load_term_at<L>(keep[q], A, b, i, ex0 + q * xstep32, ey0 + q * ystep32, true, nb);
                    scan_term<L>(sc, keep[q], track_min, with_radius);
                }
            }
        } else {
            int64_t ex = ex0, ey = ey0;
            for (int64_t i = lane; i < total; i += 32, ex += xstep32, ey += ystep32) {
                Term<L> t;
                load_term_at<L>(t, A, b, i, ex, ey, track_min, nb);
                scan_term<L>(sc, t, track_min, with_radius);
            }
        }
        const bool fb = __any_sync(0xffffffffu, sc.fb);
        const int64_t e_max = warp_max(sc.e_max);
        const int64_t e_min = warp_min(sc.e_min);
        const int64_t e_rad = warp_max(sc.e_rad);
        const uint64_t nnz = warp_sum(sc.nnz);
        const Plan pl = finish_plan(e_max, e_min, e_rad, nnz, fb, total, A.prec, A.disable_reduction);
        if (lane == g) my_pl = pl;
        if (pl.status != 0) continue;

        // ---- pass 2: accumulate
        Acc<L, NS> acc;
#pragma unroll
        for (int j = 0; j < NS; j++) acc.s[j] = 0;
        acc.err = 0;
        acc.srad = 0;
        auto do_term = [&](const Term<L>& t) {
            const bool xz = (t.kx & APB_KIND_MASK) == APB_ZERO, yz = (t.ky & APB_KIND_MASK) == APB_ZERO;
            if (!xz && !yz) acc_term<L, NS>(acc, t, pl);
            if (with_radius) rad_term<L, NS>(acc, t, pl);
        };
        if (TPL > 0) {
#pragma unroll
            for (int q = 0; q < (TPL > 0 ? TPL : 1); q++) {
                int64_t i = lane + 32 * (int64_t)q;
                if (i < total) do_term(keep[q]);
            }
        } else {
            int64_t ex = ex0, ey = ey0;
            for (int64_t i = lane; i < total; i += 32, ex += xstep32, ey += ystep32) {
                Term<L> t;
                load_term_at<L>(t, A, b, i, ex, ey, true, nb);
                do_term(t);
            }
        }

        // ---- warp reduction of (s, err, srad); s mod 2^(64 NS) with carries
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            uint64_t c = 0;
#pragma unroll
            for (int j = 0; j < NS; j++) {
                uint64_t v = __shfl_xor_sync(0xffffffffu, acc.s[j], o);
                uint64_t s1 = acc.s[j] + v;
                uint64_t c1 = s1 < v;
                uint64_t s2 = s1 + c;
                uint64_t c2 = s2 < c;
                acc.s[j] = s2;
                c = c1 | c2;
            }
            acc.err += __shfl_xor_sync(0xffffffffu, acc.err, o);
            acc.srad += __shfl_xor_sync(0xffffffffu, acc.srad, o);
        }
        if (lane == g) {
#pragma unroll
            for (int j = 0; j < NS; j++) my_s[j] = acc.s[j];
            my_err = acc.err;
            my_srad = acc.srad;
        }
    }

    // ---- parallel finalize: lane g owns dot b0 + g
    if (lane < nd) {
        const int64_t b = b0 + lane;
        if (my_pl.status != 0) {
            if (A.state) write_state(A.state + b, my_pl, 0, 0);
            if (my_pl.status == 1) {
                A.fb_flag[b] = 1;
            } else {  // ZeroResult -> Ball::zero()
                GFloat<1> z;
                z.kind = APB_ZERO;
                z.neg = 0;
                z.e = 0;
                z.n = 0;
                gf_store(A.out, b, z, mag_zero(), A.status);
            }
        } else {
            if (A.state) write_state(A.state + b, my_pl, my_err, my_srad);
            if (A.acc)
                for (int j = 0; j < my_pl.n_s && j < A.acc_stride; j++) A.acc[b * A.acc_stride + j] = my_s[j];
            finalize_store<NS>(my_pl, my_s, my_err, my_srad, A.prec, with_radius, A.out, b, A.status);
        }
    }
}

// ------------------------------------------------- lane-group kernel
// TPD lanes per dot (TPD < 32): a warp runs 32/TPD dots side by side, each
// group of TPD lanes striding over its dot's terms (lane `sub` takes terms
// sub, sub+TPD, ...), so a length-100 dot keeps every lane busy and the carry
// reduction needs log2(TPD) shuffle rounds instead of five.  A warp owns A.dpw
// dots (a multiple of 32/TPD, <= 32) processed in rounds; after each round the
// reduced state of dot g is parked in lane g, and the finalizes run on all
// lanes at the end.  Pass 2 prefetches the next term of the lane while the
// current one is accumulated.  Same arithmetic as dot_small_kernel.
// x.y term at element indices (ex, ey) of the operand arrays (no initial-value case)
template <int L>
APB_DEV void load_xy(Term<L>& t, const DotArgs& A, int64_t ex, int64_t ey, bool mant, bool neg) {
    t.kx = __ldg(A.x.kind + ex);
    t.ky = __ldg(A.y.kind + ey);
    t.ex = __ldg(A.x.exp + ex);
    t.ey = __ldg(A.y.exp + ey);
    t.rx = __ldg(A.x.rad_man + ex);
    t.ry = __ldg(A.y.rad_man + ey);
    t.fx = __ldg(A.x.rad_exp + ex);
    t.fy = __ldg(A.y.rad_exp + ey);
    if (mant) {
        if (L == 2 && A.mant16) {  // both operands 2-limb and 16-byte aligned: one vector load each
            const ulonglong2 vx = __ldg(reinterpret_cast<const ulonglong2*>(A.x.mant) + ex);
            const ulonglong2 vy = __ldg(reinterpret_cast<const ulonglong2*>(A.y.mant) + ey);
            t.xm[0] = vx.x;
            t.xm[L - 1] = vx.y;
            t.ym[0] = vy.x;
            t.ym[L - 1] = vy.y;
        } else {
            load_mant<L>(t.xm, A.x, ex);
            load_mant<L>(t.ym, A.y, ey);
        }
    }
    t.neg = neg;
}

template <int L, int NS>
APB_DEV void grp_term(Acc<L, NS>& acc, const Term<L>& t, const Plan& pl, bool with_radius) {
    const bool xz = (t.kx & APB_KIND_MASK) == APB_ZERO, yz = (t.ky & APB_KIND_MASK) == APB_ZERO;
    if (!xz && !yz) acc_term<L, NS>(acc, t, pl);
    if (with_radius) rad_term<L, NS>(acc, t, pl);
}

template <int L, int NS, int TPD>
#ifndef APB_GRP_MINB
#define APB_GRP_MINB 3  // measured on config 1: 3 blocks + one-term prefetch beat 4 and 6 without
#endif
__global__ void __launch_bounds__(128, APB_GRP_MINB) dot_grp_kernel(DotArgs A) {
    constexpr int DPR = 32 / TPD;
    constexpr int PK = NS + 7;  // parked words per dot: s[NS], err, srad, e_max, e_min, e_rad, nnz, fb
    __shared__ uint64_t park[4][32][PK];
    const int lane = threadIdx.x & 31, sub = lane % TPD, grp = lane / TPD, wl = threadIdx.x >> 5;
    const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wl;
    const int64_t b0 = warp_id * A.dpw;
    if (b0 >= A.batch) return;
    const int nd = (int)(A.batch - b0 < A.dpw ? A.batch - b0 : A.dpw);
    const int rounds = (nd + DPR - 1) / DPR;
    const bool with_radius = A.mode == APB_DOT_BALL;
    const bool track_min = A.prec > 128;
    const bool neg = A.subtract != 0;

    for (int r = 0; r < rounds; r++) {
        const int gi = r * DPR + grp;
        const bool live = gi < nd;
        const int64_t b = b0 + gi;
        int64_t ex0 = 0, xst = 0, ey0 = 0, yst = 0, nb = 0;
        if (live) dot_extent(A, b, ex0, xst, ey0, yst, nb);
        const int64_t total = live ? nb + (A.has_init ? 1 : 0) : 0;
        const bool init_lane = live && A.has_init && sub == 0;
        ex0 += sub * xst;
        ey0 += sub * yst;
        const int64_t xstp = TPD * xst, ystp = TPD * yst;
        // ---- pass 1: setup scan (metadata only unless e_min is tracked)
        ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
        {
            constexpr int SB = 2;  // terms per lane with loads in flight together
            int64_t ex = ex0, ey = ey0;
            for (int64_t i0 = sub; i0 < nb; i0 += SB * TPD, ex += SB * xstp, ey += SB * ystp) {
                Term<L> t[SB];
#pragma unroll
                for (int q = 0; q < SB; q++)
                    if (i0 + q * TPD < nb) load_xy<L>(t[q], A, ex + q * xstp, ey + q * ystp, track_min, neg);
#pragma unroll
                for (int q = 0; q < SB; q++)
                    if (i0 + q * TPD < nb) scan_term<L>(sc, t[q], track_min, with_radius);
            }
            if (init_lane) {
                Term<L> t;
                load_term_at<L>(t, A, b, nb, 0, 0, true, nb);
                scan_term<L>(sc, t, track_min, with_radius);
            }
        }
#pragma unroll
        for (int o = TPD / 2; o; o >>= 1) {
            int64_t v = __shfl_xor_sync(0xffffffffu, sc.e_max, o);
            sc.e_max = v > sc.e_max ? v : sc.e_max;
            v = __shfl_xor_sync(0xffffffffu, sc.e_min, o);
            sc.e_min = v < sc.e_min ? v : sc.e_min;
            v = __shfl_xor_sync(0xffffffffu, sc.e_rad, o);
            sc.e_rad = v > sc.e_rad ? v : sc.e_rad;
            sc.nnz += __shfl_xor_sync(0xffffffffu, sc.nnz, o);
            sc.fb |= __shfl_xor_sync(0xffffffffu, (int)sc.fb, o) != 0;
        }
        const Plan pl = finish_plan(sc.e_max, sc.e_min, sc.e_rad, sc.nnz, sc.fb, total, A.prec, A.disable_reduction);

        // ---- pass 2: accumulate (the group's plan is uniform across its lanes)
        Acc<L, NS> acc;
#pragma unroll
        for (int j = 0; j < NS; j++) acc.s[j] = 0;
        acc.err = 0;
        acc.srad = 0;
        if (live && pl.status == 0) {
            int64_t ex = ex0, ey = ey0;
            Term<L> cur;
#ifndef APB_GRP_PREFETCH
#define APB_GRP_PREFETCH 1
#endif
#if APB_GRP_PREFETCH == 2
            Term<L> cur1;
            if (sub < nb) load_xy<L>(cur, A, ex, ey, true, neg);
            if (sub + TPD < nb) load_xy<L>(cur1, A, ex + xstp, ey + ystp, true, neg);
            ex += 2 * xstp;
            ey += 2 * ystp;
            for (int64_t i = sub; i < nb; i += TPD, ex += xstp, ey += ystp) {
                Term<L> nxt;
                if (i + 2 * TPD < nb) load_xy<L>(nxt, A, ex, ey, true, neg);
                grp_term<L, NS>(acc, cur, pl, with_radius);
                cur = cur1;
                cur1 = nxt;
            }
#elif APB_GRP_PREFETCH
            if (sub < nb) load_xy<L>(cur, A, ex, ey, true, neg);
            for (int64_t i = sub; i < nb; i += TPD) {
                ex += xstp;
                ey += ystp;
                Term<L> nxt;
                if (i + TPD < nb) load_xy<L>(nxt, A, ex, ey, true, neg);
                grp_term<L, NS>(acc, cur, pl, with_radius);
                cur = nxt;
            }
#else
            for (int64_t i = sub; i < nb; i += TPD, ex += xstp, ey += ystp) {
                load_xy<L>(cur, A, ex, ey, true, neg);
                grp_term<L, NS>(acc, cur, pl, with_radius);
            }
#endif
            if (init_lane) {
                load_term_at<L>(cur, A, b, nb, 0, 0, true, nb);
                grp_term<L, NS>(acc, cur, pl, with_radius);
            }
        }
        // ---- group reduction of (s, err, srad) mod 2^(64 NS)
#pragma unroll
        for (int o = TPD / 2; o; o >>= 1) {
            uint64_t c = 0;
#pragma unroll
            for (int j = 0; j < NS; j++) {
                const uint64_t v = __shfl_xor_sync(0xffffffffu, acc.s[j], o);
                const uint64_t s1 = acc.s[j] + v;
                const uint64_t c1 = s1 < v;
                const uint64_t s2 = s1 + c;
                acc.s[j] = s2;
                c = c1 | (s2 < c);
            }
            acc.err += __shfl_xor_sync(0xffffffffu, acc.err, o);
            acc.srad += __shfl_xor_sync(0xffffffffu, acc.srad, o);
        }
        // ---- park dot gi's state (group leader) for the parallel finalize
        if (live && sub == 0) {
            uint64_t* pk = park[wl][gi];
#pragma unroll
            for (int j = 0; j < NS; j++) pk[j] = acc.s[j];
            pk[NS] = acc.err;
            pk[NS + 1] = acc.srad;
            pk[NS + 2] = (uint64_t)sc.e_max;
            pk[NS + 3] = (uint64_t)sc.e_min;
            pk[NS + 4] = (uint64_t)sc.e_rad;
            pk[NS + 5] = sc.nnz;
            pk[NS + 6] = sc.fb ? 1 : 0;
        }
    }
    __syncwarp();

    // ---- parallel finalize: lane g owns dot b0 + g
    if (lane < nd) {
        const int64_t b = b0 + lane;
        const uint64_t* pk = park[wl][lane];
        int64_t ex0, xst, ey0, yst, nb;
        dot_extent(A, b, ex0, xst, ey0, yst, nb);
        const int64_t total = nb + (A.has_init ? 1 : 0);
        const Plan pl = finish_plan((int64_t)pk[NS + 2], (int64_t)pk[NS + 3], (int64_t)pk[NS + 4], pk[NS + 5],
                                    pk[NS + 6] != 0, total, A.prec, A.disable_reduction);
        if (pl.status != 0) {
            if (A.state) write_state(A.state + b, pl, 0, 0);
            if (pl.status == 1) {
                A.fb_flag[b] = 1;
            } else {
                GFloat<1> z;
                z.kind = APB_ZERO;
                z.neg = 0;
                z.e = 0;
                z.n = 0;
                gf_store(A.out, b, z, mag_zero(), A.status);
            }
        } else {
            uint64_t s[NS];
#pragma unroll
            for (int j = 0; j < NS; j++) s[j] = pk[j];
            if (A.state) write_state(A.state + b, pl, pk[NS], pk[NS + 1]);
            if (A.acc)
                for (int j = 0; j < pl.n_s && j < A.acc_stride; j++) A.acc[b * A.acc_stride + j] = s[j];
            finalize_store<NS>(pl, s, pk[NS], pk[NS + 1], A.prec, with_radius, A.out, b, A.status);
        }
    }
}

#include "dot_reg.cuh"

// ------------------------------------------------- bulk-staged kernel
// Contiguous batches (dot b = elements [b n, (b+1) n) of x and y, n even, 2-limb
// operands, 16-byte aligned arrays -- config 1): a persistent CTA of 8 warps
// streams chunks of 8 consecutive dots through a 3-stage shared-memory ring with
// cp.async.bulk (10 bulk copies per chunk: the five SoA arrays of x and y, each
// one contiguous range), so the memory system always has ~2 chunks per SM in
// flight without holding registers.  Warp w takes dot w of the chunk: lanes over
// its terms, both passes read shared memory; the reduced states are parked per
// warp and finalized 32 at a time, one dot per lane.  Arithmetic = dot_small.
#ifndef APB_BLK_DOTS
#define APB_BLK_DOTS 16
#endif
#ifndef APB_BLK_STAGES
#define APB_BLK_STAGES 1
#endif
constexpr int BLK_DOTS = APB_BLK_DOTS, BLK_STAGES = APB_BLK_STAGES;  // dots (= warps) per chunk, ring depth

struct BlkLayout {  // byte offsets of one stage (16-byte aligned pieces)
    int xm, ym, xe, ye, xf, yf, xr, yr, xk, yk, bytes;
};
__host__ __device__ inline int align16(int v) { return (v + 15) & ~15; }
__host__ __device__ inline BlkLayout blk_layout(int n, int L) {
    BlkLayout o;
    const int E = BLK_DOTS * n;
    int off = 0;
    o.xm = off; off += align16(E * L * 8);
    o.ym = off; off += align16(E * L * 8);
    o.xe = off; off += align16(E * 8);
    o.ye = off; off += align16(E * 8);
    o.xf = off; off += align16(E * 8);
    o.yf = off; off += align16(E * 8);
    o.xr = off; off += align16(E * 4);
    o.yr = off; off += align16(E * 4);
    o.xk = off; off += align16(E);
    o.yk = off; off += align16(E);
    o.bytes = off;
    return o;
}

APB_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
APB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
APB_DEV void mbar_init1(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
}
APB_DEV void mbar_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
APB_DEV void mbar_wait_par(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n"
        "}\n" ::"r"(smem_addr(bar)),
        "r"(parity)
        : "memory");
}

template <int L>
APB_DEV void blk_issue(uint8_t* st, uint64_t* bar, const DotArgs& A, const BlkLayout& lay, int64_t chunk, int n) {
    const int64_t d0 = chunk * BLK_DOTS;
    const int nd = (int)(A.batch - d0 < BLK_DOTS ? A.batch - d0 : BLK_DOTS);
    const int64_t ex = A.idx.x_off + d0 * n, ey = A.idx.y_off + d0 * n;
    const uint32_t E = (uint32_t)(nd * n);
    mbar_expect(bar, E * (2 * (L * 8 + 8 + 8 + 4 + 1)));
    bulk_g2s(st + lay.xm, A.x.mant + ex * L, E * L * 8, bar);
    bulk_g2s(st + lay.ym, A.y.mant + ey * L, E * L * 8, bar);
    bulk_g2s(st + lay.xe, A.x.exp + ex, E * 8, bar);
    bulk_g2s(st + lay.ye, A.y.exp + ey, E * 8, bar);
    bulk_g2s(st + lay.xf, A.x.rad_exp + ex, E * 8, bar);
    bulk_g2s(st + lay.yf, A.y.rad_exp + ey, E * 8, bar);
    bulk_g2s(st + lay.xr, A.x.rad_man + ex, E * 4, bar);
    bulk_g2s(st + lay.yr, A.y.rad_man + ey, E * 4, bar);
    bulk_g2s(st + lay.xk, A.x.kind + ex, E, bar);
    bulk_g2s(st + lay.yk, A.y.kind + ey, E, bar);
}

template <int L>
APB_DEV void blk_term(Term<L>& t, const uint8_t* st, const BlkLayout& lay, int e, bool neg, bool mant) {
    t.kx = st[lay.xk + e];
    t.ky = st[lay.yk + e];
    t.ex = ((const int64_t*)(st + lay.xe))[e];
    t.ey = ((const int64_t*)(st + lay.ye))[e];
    t.fx = ((const int64_t*)(st + lay.xf))[e];
    t.fy = ((const int64_t*)(st + lay.yf))[e];
    t.rx = ((const uint32_t*)(st + lay.xr))[e];
    t.ry = ((const uint32_t*)(st + lay.yr))[e];
    if (mant) {
#pragma unroll
        for (int j = 0; j < L; j++) {
            t.xm[j] = ((const uint64_t*)(st + lay.xm))[e * L + j];
            t.ym[j] = ((const uint64_t*)(st + lay.ym))[e * L + j];
        }
    }
    t.neg = neg;
}

template <int L, int NS>
__global__ void __launch_bounds__(32 * BLK_DOTS, 1) dot_blk_kernel(DotArgs A, int64_t nchunks) {
    extern __shared__ __align__(128) uint8_t blk_smem[];
    constexpr int PK = NS + 8;  // s[NS], err, srad, e_max, e_min, e_rad, nnz, fb, dot index
    const int n = (int)A.n;
    const BlkLayout lay = blk_layout(n, L);
    uint8_t* stages = blk_smem;
    uint64_t* bars = (uint64_t*)(blk_smem + BLK_STAGES * lay.bytes);
    uint64_t* park = bars + BLK_STAGES;  // [warps][32][PK]
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t* mypark = park + (size_t)w * 32 * PK;
    const bool with_radius = A.mode == APB_DOT_BALL;
    const bool track_min = A.prec > 128;
    const bool neg = A.subtract != 0;
    if (threadIdx.x == 0) {
        for (int q = 0; q < BLK_STAGES; q++) mbar_init1(&bars[q]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    // this CTA's chunks: blockIdx.x + k * gridDim.x
    const int64_t my_n = nchunks > blockIdx.x ? (nchunks - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    if (threadIdx.x == 0)
        for (int64_t k = 0; k < BLK_STAGES - 1 && k < my_n; k++)
            blk_issue<L>(stages + k * lay.bytes, &bars[k], A, lay, blockIdx.x + k * gridDim.x, n);
    int parked = 0;
    for (int64_t k = 0; k < my_n; k++) {
        __syncthreads();  // every warp is done with chunk k-1: its stage is free
        if (threadIdx.x == 0 && k + BLK_STAGES - 1 < my_n) {
            const int64_t kk = k + BLK_STAGES - 1;
            blk_issue<L>(stages + (kk % BLK_STAGES) * lay.bytes, &bars[kk % BLK_STAGES], A, lay,
                         blockIdx.x + kk * gridDim.x, n);
        }
        const int sidx = (int)(k % BLK_STAGES);
        mbar_wait_par(&bars[sidx], (uint32_t)((k / BLK_STAGES) & 1));
        const uint8_t* st = stages + sidx * lay.bytes;
        const int64_t chunk = blockIdx.x + k * gridDim.x;
        const int64_t b = chunk * BLK_DOTS + w;
        if (b < A.batch) {
            const int e0 = w * n;
            ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
            for (int i = lane; i < n; i += 32) {
                Term<L> t;
                blk_term<L>(t, st, lay, e0 + i, neg, track_min);
                scan_term<L>(sc, t, track_min, with_radius);
            }
            const bool fb = __any_sync(0xffffffffu, sc.fb);
            sc.e_max = warp_max(sc.e_max);
            sc.e_min = warp_min(sc.e_min);
            sc.e_rad = warp_max(sc.e_rad);
            sc.nnz = warp_sum(sc.nnz);
            const Plan pl = finish_plan(sc.e_max, sc.e_min, sc.e_rad, sc.nnz, fb, n, A.prec, A.disable_reduction);
            Acc<L, NS> acc;
#pragma unroll
            for (int j = 0; j < NS; j++) acc.s[j] = 0;
            acc.err = 0;
            acc.srad = 0;
            if (pl.status == 0) {
                for (int i = lane; i < n; i += 32) {
                    Term<L> t;
                    blk_term<L>(t, st, lay, e0 + i, neg, true);
                    const bool xz = (t.kx & APB_KIND_MASK) == APB_ZERO, yz = (t.ky & APB_KIND_MASK) == APB_ZERO;
                    if (!xz && !yz) acc_term<L, NS>(acc, t, pl);
                    if (with_radius) rad_term<L, NS>(acc, t, pl);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                uint64_t c = 0;
#pragma unroll
                for (int j = 0; j < NS; j++) {
                    const uint64_t v = __shfl_xor_sync(0xffffffffu, acc.s[j], o);
                    const uint64_t s1 = acc.s[j] + v;
                    const uint64_t c1 = s1 < v;
                    const uint64_t s2 = s1 + c;
                    acc.s[j] = s2;
                    c = c1 | (s2 < c);
                }
                acc.err += __shfl_xor_sync(0xffffffffu, acc.err, o);
                acc.srad += __shfl_xor_sync(0xffffffffu, acc.srad, o);
            }
            if (lane == 0) {
                uint64_t* pk = mypark + (size_t)parked * PK;
#pragma unroll
                for (int j = 0; j < NS; j++) pk[j] = acc.s[j];
                pk[NS] = acc.err;
                pk[NS + 1] = acc.srad;
                pk[NS + 2] = (uint64_t)sc.e_max;
                pk[NS + 3] = (uint64_t)sc.e_min;
                pk[NS + 4] = (uint64_t)sc.e_rad;
                pk[NS + 5] = sc.nnz;
                pk[NS + 6] = fb ? 1 : 0;
                pk[NS + 7] = (uint64_t)b;
            }
            parked++;
        }
        // finalize 32 parked dots (or the rest at the end), one per lane
        if (parked == 32 || (k + 1 == my_n && parked > 0)) {
            __syncwarp();
            if (lane < parked) {
                const uint64_t* pk = mypark + (size_t)lane * PK;
                const int64_t bb = (int64_t)pk[NS + 7];
                const Plan pl = finish_plan((int64_t)pk[NS + 2], (int64_t)pk[NS + 3], (int64_t)pk[NS + 4], pk[NS + 5],
                                            pk[NS + 6] != 0, n, A.prec, A.disable_reduction);
                if (pl.status != 0) {
                    if (A.state) write_state(A.state + bb, pl, 0, 0);
                    if (pl.status == 1) {
                        A.fb_flag[bb] = 1;
                    } else {
                        GFloat<1> z;
                        z.kind = APB_ZERO;
                        z.neg = 0;
                        z.e = 0;
                        z.n = 0;
                        gf_store(A.out, bb, z, mag_zero(), A.status);
                    }
                } else {
                    uint64_t sv[NS];
#pragma unroll
                    for (int j = 0; j < NS; j++) sv[j] = pk[j];
                    if (A.state) write_state(A.state + bb, pl, pk[NS], pk[NS + 1]);
                    if (A.acc)
                        for (int j = 0; j < pl.n_s && j < A.acc_stride; j++) A.acc[bb * A.acc_stride + j] = sv[j];
                    finalize_store<NS>(pl, sv, pk[NS], pk[NS + 1], A.prec, with_radius, A.out, bb, A.status);
                }
            }
            __syncwarp();
            parked = 0;
        }
    }
}

// eligibility: contiguous dots of even length n, equal 2-limb x / y, 16-byte
// aligned arrays and offsets, no initial value, stage fits shared memory
static bool blk_ok(const DotArgs& A, int L) {
    // opt-in (APB_DOT_BULK=1): measured compute-bound at 0.24-0.30 ms on config 1
    // against 0.234 ms for dot_grp_kernel, whose lane groups need fewer instructions
    static const bool on = std::getenv("APB_DOT_BULK") != nullptr;
    if (!on || A.palen > 0 || A.has_init || A.n <= 0 || ((BLK_DOTS * A.n) & 15) || A.x.L != L || A.y.L != L)
        return false;  // (chunk offsets of the 1-byte kind arrays stay 16-byte aligned)
    if (A.idx.xstep != 1 || A.idx.ystep != 1 || A.idx.xs1 != A.n || A.idx.ys1 != A.n) return false;
    if (A.idx.bdiv != 1 && (A.idx.xs2 != 0 || A.idx.ys2 != 0)) return false;
    if ((A.idx.x_off & 15) || (A.idx.y_off & 15)) return false;
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (!al(A.x.mant) || !al(A.x.exp) || !al(A.x.kind) || !al(A.x.rad_man) || !al(A.x.rad_exp)) return false;
    if (!al(A.y.mant) || !al(A.y.exp) || !al(A.y.kind) || !al(A.y.rad_man) || !al(A.y.rad_exp)) return false;
    const BlkLayout lay = blk_layout((int)A.n, L);
    return (size_t)BLK_STAGES * lay.bytes + 64 + (size_t)BLK_DOTS * 32 * 16 * 8 <= 225 * 1024;
}

template <int L, int NS>
static void launch_blk(const DotArgs& A, cudaStream_t st) {
    constexpr int PK = NS + 8;
    const BlkLayout lay = blk_layout((int)A.n, L);
    const size_t shm = (size_t)BLK_STAGES * lay.bytes + BLK_STAGES * 8 + (size_t)BLK_DOTS * 32 * PK * 8;
    static size_t attr = 0;
    if (shm > attr) {
        cudaFuncSetAttribute(dot_blk_kernel<L, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        attr = shm;
    }
    const int64_t nchunks = (A.batch + BLK_DOTS - 1) / BLK_DOTS;
    const unsigned grid = (unsigned)std::min<int64_t>(nchunks, 148);
    dot_blk_kernel<L, NS><<<grid, 32 * BLK_DOTS, shm, st>>>(A, nchunks);
    count_launch();
}

// ------------------------------------------------- staged small kernel
// For dots of <= 128 terms with <= 2-limb operands (config 1): the warp's 32
// dots are software-pipelined through shared memory -- while dot g is
// scanned and accumulated from its stage, cp.async copies of dot g+1's
// mantissas, exponents and radii land in the other stage (kind bytes are
// prefetched into registers).  Each lane only touches its own term slots, so
// no barrier is needed beyond cp.async.wait_group.
constexpr int STG_T = 128;  // term slots per stage (4 per lane)

template <int L>
struct StageBuf {
    uint64_t xm[L][STG_T], ym[L][STG_T];
    int64_t xe[STG_T], ye[STG_T], xf[STG_T], yf[STG_T];
    uint32_t xr[STG_T], yr[STG_T];
};

APB_DEV void cp_async(void* sdst, const void* gsrc, int bytes) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
    if (bytes == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
    else if (bytes == 8)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
APB_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
APB_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// issue the copies of dot b's terms (this lane's slots) into stage buf; return kinds
template <int L>
APB_DEV void stage_dot(StageBuf<L>& sb, uint32_t (&kinds)[4], const DotArgs& A, int64_t b, int64_t total,
                       int lane) {
    const int64_t bq = A.idx.bdiv == 1 ? b : b / A.idx.bdiv;
    const int64_t br = A.idx.bdiv == 1 ? 0 : b - bq * A.idx.bdiv;
    const int64_t xb = A.idx.x_off + bq * A.idx.xs1 + br * A.idx.xs2;
    const int64_t yb = A.idx.y_off + bq * A.idx.ys1 + br * A.idx.ys2;
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int64_t i = lane + 32 * q;
        const int slot = lane + 32 * q;
        kinds[q] = 0;
        if (i >= total) continue;
        const BallsView& X = i < A.n ? A.x : A.init;
        const int64_t ex = i < A.n ? xb + i * A.idx.xstep : b;
        // x operand (or the initial value)
        const int offx = L - X.L;
#pragma unroll
        for (int j = 0; j < L; j++) {
            if (j >= offx) cp_async(&sb.xm[j][slot], X.mant + ex * X.L + (j - offx), 8);
            else sb.xm[j][slot] = 0;
        }
        cp_async(&sb.xe[slot], X.exp + ex, 8);
        cp_async(&sb.xf[slot], X.rad_exp + ex, 8);
        cp_async(&sb.xr[slot], X.rad_man + ex, 4);
        uint32_t kx = __ldg(X.kind + ex), ky = APB_FINITE;
        if (i < A.n) {
            const int64_t ey = yb + i * A.idx.ystep;
            const int offy = L - A.y.L;
#pragma unroll
            for (int j = 0; j < L; j++) {
                if (j >= offy) cp_async(&sb.ym[j][slot], A.y.mant + ey * A.y.L + (j - offy), 8);
                else sb.ym[j][slot] = 0;
            }
            cp_async(&sb.ye[slot], A.y.exp + ey, 8);
            cp_async(&sb.yf[slot], A.y.rad_exp + ey, 8);
            cp_async(&sb.yr[slot], A.y.rad_man + ey, 4);
            ky = __ldg(A.y.kind + ey);
        } else {  // y = 1 for the initial term
#pragma unroll
            for (int j = 0; j < L; j++) sb.ym[j][slot] = (j == L - 1) ? (1ull << 63) : 0ull;
            sb.ye[slot] = 1;
            sb.yf[slot] = 0;
            sb.yr[slot] = 0;
        }
        kinds[q] = kx | (ky << 8);
    }
}

template <int L>
APB_DEV void read_term(Term<L>& t, const StageBuf<L>& sb, int slot, uint32_t kinds, bool sub) {
#pragma unroll
    for (int j = 0; j < L; j++) {
        t.xm[j] = sb.xm[j][slot];
        t.ym[j] = sb.ym[j][slot];
    }
    t.ex = sb.xe[slot];
    t.ey = sb.ye[slot];
    t.fx = sb.xf[slot];
    t.fy = sb.yf[slot];
    t.rx = sb.xr[slot];
    t.ry = sb.yr[slot];
    t.kx = (uint8_t)(kinds & 255u);
    t.ky = (uint8_t)(kinds >> 8);
    t.neg = sub;
}

template <int L, int NS>
__global__ void __launch_bounds__(128, 3) dot_staged_kernel(DotArgs A) {
    extern __shared__ __align__(16) uint8_t stg_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    StageBuf<L>* bufs = reinterpret_cast<StageBuf<L>*>(stg_raw) + 2 * wl;
    const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wl;
    const int64_t b0 = warp_id * 32;
    if (b0 >= A.batch) return;
    const int nd = (int)(A.batch - b0 < 32 ? A.batch - b0 : 32);
    const int64_t total = A.n + (A.has_init ? 1 : 0);
    const bool with_radius = A.mode == APB_DOT_BALL;
    const bool track_min = A.prec > 128;

    Plan my_pl;
    uint64_t my_s[NS];
    uint64_t my_err = 0, my_srad = 0;
    my_pl.status = 2;

    uint32_t kinds[4], kinds_next[4];
    stage_dot<L>(bufs[0], kinds, A, b0, total, lane);
    cp_commit();
    for (int g = 0; g < nd; g++) {
        const int64_t b = b0 + g;
        if (g + 1 < nd) {
            stage_dot<L>(bufs[(g + 1) & 1], kinds_next, A, b + 1, total, lane);
            cp_commit();
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        const StageBuf<L>& sb = bufs[g & 1];
        // ---- pass 1: setup scan from the stage
        ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t i = lane + 32 * q;
            if (i < total) {
                Term<L> t;
                read_term<L>(t, sb, lane + 32 * q, kinds[q], (i < A.n) && A.subtract);
                scan_term<L>(sc, t, track_min, with_radius);
            }
        }
        const bool fb = __any_sync(0xffffffffu, sc.fb);
        const int64_t e_max = warp_max(sc.e_max);
        const int64_t e_min = warp_min(sc.e_min);
        const int64_t e_rad = warp_max(sc.e_rad);
        const uint64_t nnz = warp_sum(sc.nnz);
        const Plan pl = finish_plan(e_max, e_min, e_rad, nnz, fb, total, A.prec, A.disable_reduction);
        if (lane == g) my_pl = pl;
        if (pl.status == 0) {
            Acc<L, NS> acc;
#pragma unroll
            for (int j = 0; j < NS; j++) acc.s[j] = 0;
            acc.err = 0;
            acc.srad = 0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const int64_t i = lane + 32 * q;
                if (i < total) {
                    Term<L> t;
                    read_term<L>(t, sb, lane + 32 * q, kinds[q], (i < A.n) && A.subtract);
                    const bool xz = (t.kx & APB_KIND_MASK) == APB_ZERO, yz = (t.ky & APB_KIND_MASK) == APB_ZERO;
                    if (!xz && !yz) acc_term<L, NS>(acc, t, pl);
                    if (with_radius) rad_term<L, NS>(acc, t, pl);
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                uint64_t c = 0;
#pragma unroll
                for (int j = 0; j < NS; j++) {
                    uint64_t v = __shfl_xor_sync(0xffffffffu, acc.s[j], o);
                    uint64_t s1 = acc.s[j] + v;
                    uint64_t c1 = s1 < v;
                    uint64_t s2 = s1 + c;
                    uint64_t c2 = s2 < c;
                    acc.s[j] = s2;
                    c = c1 | c2;
                }
                acc.err += __shfl_xor_sync(0xffffffffu, acc.err, o);
                acc.srad += __shfl_xor_sync(0xffffffffu, acc.srad, o);
            }
            if (lane == g) {
#pragma unroll
                for (int j = 0; j < NS; j++) my_s[j] = acc.s[j];
                my_err = acc.err;
                my_srad = acc.srad;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) kinds[q] = kinds_next[q];
    }

    if (lane < nd) {
        const int64_t b = b0 + lane;
        if (my_pl.status != 0) {
            if (A.state) write_state(A.state + b, my_pl, 0, 0);
            if (my_pl.status == 1) {
                A.fb_flag[b] = 1;
            } else {
                GFloat<1> z;
                z.kind = APB_ZERO;
                z.neg = 0;
                z.e = 0;
                z.n = 0;
                gf_store(A.out, b, z, mag_zero(), A.status);
            }
        } else {
            if (A.state) write_state(A.state + b, my_pl, my_err, my_srad);
            if (A.acc)
                for (int j = 0; j < my_pl.n_s && j < A.acc_stride; j++) A.acc[b * A.acc_stride + j] = my_s[j];
            finalize_store<NS>(my_pl, my_s, my_err, my_srad, A.prec, with_radius, A.out, b, A.status);
        }
    }
}

// ====================================================== generic (thread/dot)

APB_DEV Mag mag_upper_of(const GF& x) {
    if (x.kind == APB_ZERO) return mag_zero();
    // the reference reads an empty limb vector here (unspecified); an infinite
    // midpoint has an infinite magnitude bound
    if (x.kind != APB_FINITE) return mag_inf();
    return mag_parts((x.d[x.n - 1] >> 34) + 1, x.e);
}

struct GBall {
    GF m;
    Mag r;
};

__device__ void gb_load(GBall& g, const BallsView& a, int64_t e) {
    gf_load(g.m, a, e);
    g.r = mag_load(a.rad_man[e], a.rad_exp[e]);
}

__device__ void gb_one(GBall& g) {
    g.m.kind = APB_FINITE;
    g.m.neg = 0;
    g.m.e = 1;
    g.m.n = 1;
    g.m.d[0] = 1ull << 63;
    g.r = mag_zero();
}

__device__ void gf_negate(GF& x) {
    if (x.kind == APB_FINITE) x.neg = !x.neg;
    else if (x.kind == APB_PINF) {
        x.kind = APB_NINF;
        x.neg = 1;
    } else if (x.kind == APB_NINF) {
        x.kind = APB_PINF;
        x.neg = 0;
    }
}

// ball_fallback_addmul (src/ball.cpp:21-36), acc updated in place
__device__ void gb_addmul(GBall& acc, const GBall& x, const GBall& y, int64_t p, GF& tmp, int* status) {
    if (acc.m.kind == APB_NAN || x.m.kind == APB_NAN || y.m.kind == APB_NAN) {
        acc.m.kind = APB_NAN;
        acc.m.n = 0;
        acc.r = mag_inf();
        return;
    }
    gf_mul_exact(tmp, x.m, y.m, status);
    if (tmp.kind == APB_NAN) {
        acc.m.kind = APB_NAN;
        acc.m.n = 0;
        acc.r = mag_inf();
        return;
    }
    Mag rad = acc.r;
    if (y.r.kind != 0 && x.m.kind != APB_ZERO) rad = mag_add(rad, mag_mul(mag_upper_of(x.m), y.r));
    if (x.r.kind != 0 && y.m.kind != APB_ZERO) rad = mag_add(rad, mag_mul(mag_upper_of(y.m), x.r));
    if (x.r.kind != 0 && y.r.kind != 0) rad = mag_add(rad, mag_mul(x.r, y.r));
    Mag perr = gf_round(tmp, p, status);
    Mag aerr = gf_add_round(acc.m, acc.m, tmp, p, status);
    if (acc.m.kind == APB_NAN) {
        acc.r = mag_inf();
        return;
    }
    acc.r = mag_add(rad, mag_add(perr, aerr));
}

// Column-wise ("comba") exact sum of the partial products a_i b_j with i + j >= base,
// each placed at limb i + j - base of a wlen-limb result: every output limb is
// written once (three-word running column sum), no read-modify-write of a
// local-memory product array.  With base = 0 this is the full product; with the
// base of mulhigh_approx it is exactly the window that routine accumulates (the
// same pairs, full 128-bit products, exact carries), so both agree bit for bit.
__device__ void g_comba(const uint64_t* a, int na, const uint64_t* b, int nb, int base, uint64_t* out, int wlen) {
    uint64_t c0 = 0, c1 = 0, c2 = 0;
    for (int c = 0; c < wlen; c++) {
        const int col = c + base;  // i + j
        const int ilo = col - (nb - 1) > 0 ? col - (nb - 1) : 0;
        const int ihi = col < na - 1 ? col : na - 1;
        for (int i = ilo; i <= ihi; i++) {
            uint64_t lo, hi;
            mul64(a[i], b[col - i], lo, hi);
            c0 += lo;
            const uint64_t k0 = c0 < lo;
            const uint64_t h = hi + k0;  // hi <= 2^64 - 2: no wrap
            c1 += h;
            c2 += c1 < h;
        }
        out[c] = c0;
        c0 = c1;
        c1 = c2;
        c2 = 0;
    }
}

// mulhigh_approx (include/apball/limb.hpp:194-228)
__device__ void g_mulhigh(const uint64_t* a, int na, const uint64_t* b, int nb, int k, uint64_t* out) {
    const int total = na + nb;
    const int base = total - k >= 2 ? total - k - 2 : 0;
    const int wlen = total - base;
    uint64_t w[2 * GCAP];
    g_comba(a, na, b, nb, base, w, wlen);
    for (int i = 0; i < k; i++) out[i] = w[wlen - k + i];
}

// accumulate_aligned (src/dot.cpp:139-173) on a runtime-size accumulator
__device__ void g_acc_aligned(const Plan& pl, uint64_t* s, uint64_t& err, const uint64_t* t, int nt,
                              int64_t e_term, bool negate) {
    const int64_t shift = pl.e_s - e_term;
    if (shift >= 64 * (int64_t)pl.n_s) {
        err++;
        return;
    }
    const unsigned sb = (unsigned)(shift % 64);
    const int sl = (int)(shift / 64);
    uint64_t buf[2 * GCAP + 2];
    if (sb) {
        buf[0] = t[0] << (64 - sb);
        for (int i = 0; i + 1 < nt; i++) buf[i + 1] = (t[i] >> sb) | (t[i + 1] << (64 - sb));
        buf[nt] = t[nt - 1] >> sb;
        t = buf;
        nt++;
    }
    while (nt && t[0] == 0) {
        t++;
        nt--;
    }
    if (nt == 0) return;
    const int avail = pl.n_s - sl;
    int ds, dt, v;
    if (nt <= avail) {
        ds = avail - nt;
        dt = 0;
        v = nt;
    } else {
        ds = 0;
        dt = nt - avail;
        v = avail;
        err++;
    }
    uint64_t* w = s + ds;
    if (!negate) {
        uint64_t c = 0;
        for (int i = 0; i < v; i++) {
            uint64_t y = t[dt + i];
            uint64_t s1 = w[i] + y;
            uint64_t c1 = s1 < y;
            uint64_t s2 = s1 + c;
            c = c1 | (s2 < c);
            w[i] = s2;
        }
        for (int i = v; ds + i < pl.n_s && c; i++) {
            uint64_t s1 = w[i] + c;
            c = s1 < c;
            w[i] = s1;
        }
    } else {
        uint64_t bw = 0;
        for (int i = 0; i < v; i++) {
            uint64_t x = w[i], y = t[dt + i];
            w[i] = x - y - bw;
            bw = (x < y) || (x == y && bw);
        }
        for (int i = v; ds + i < pl.n_s && bw; i++) {
            uint64_t x = w[i];
            w[i] = x - 1;
            bw = x == 0;
        }
    }
}

// general dot_accumulate_term (src/dot.cpp:229-273) incl. truncation and mulhigh
__device__ void g_acc_term(const Plan& pl, uint64_t* s, uint64_t& err, const GF& m, const GF& mp,
                           bool negate) {
    negate ^= (m.neg != 0) ^ (mp.neg != 0);
    const int64_t e_term = m.e + mp.e;
    const int64_t shift = pl.e_s - e_term;
    if (shift >= 64 * (int64_t)pl.n_s) {
        err++;
        return;
    }
    const int n = m.n, np = mp.n;
    const int64_t p_t = 64 * (int64_t)pl.n_s - shift;
    const int ncap = (int)((p_t + 63) / 64) + 1;
    const int na = n < ncap ? n : ncap, nb = np < ncap ? np : ncap;
    if (n > ncap || np > ncap) err++;
    const uint64_t* a = m.d + (n - na);
    const uint64_t* bb = mp.d + (np - nb);
    const int nt = na + nb;
    uint64_t t[2 * GCAP];
    int lead = nt;
    bool short_prod = false;
    const int mn = n < np ? n : np;
    if (p_t >= 25 * 64 && 640 * (int64_t)mn > 9 * p_t) {
        const int v = pl.n_s - (int)(shift / 64);
        const int k = nt < v + 1 ? nt : v + 1;
        if (k < nt) {
            g_mulhigh(a, na, bb, nb, k, t);
            err++;
            lead = k;
            short_prod = true;
        }
    }
    if (!short_prod) g_comba(a, na, bb, nb, 0, t, nt);  // full product, column-wise
    g_acc_aligned(pl, s, err, t, lead, e_term, negate);
}

// setup_core over term i via a callback that yields (x, y, neg)
template <class GetTerm>
__device__ Plan g_setup(GetTerm&& get, int64_t total, int64_t p, bool with_radius, bool disable_red,
                        GBall& xs, GBall& ys) {
    ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
    const bool track_min = p > 128;
    for (int64_t i = 0; i < total && !sc.fb; i++) {
        bool neg;
        get(i, xs, ys, neg);
        const GF& xm = xs.m;
        const GF& ym = ys.m;
        const bool xf = xm.kind == APB_ZERO || xm.kind == APB_FINITE;
        const bool yf = ym.kind == APB_ZERO || ym.kind == APB_FINITE;
        if (!xf || !yf) {
            sc.fb = true;
            break;
        }
        if ((xm.kind != APB_ZERO && exp_huge(xm.e)) || (ym.kind != APB_ZERO && exp_huge(ym.e))) {
            sc.fb = true;
            break;
        }
        if (xm.kind != APB_ZERO && ym.kind != APB_ZERO) {
            sc.nnz++;
            int64_t ee = xm.e + ym.e;
            if (ee > sc.e_max) sc.e_max = ee;
            if (track_min) {
                int64_t lo = ee - 64 * (int64_t)(xm.n + ym.n);
                if (lo < sc.e_min) sc.e_min = lo;
            }
        }
        if (with_radius) {
            const Mag& xr = xs.r;
            const Mag& yr = ys.r;
            if (xr.kind == 2 || yr.kind == 2 || (xr.kind == 1 && exp_huge(xr.f)) ||
                (yr.kind == 1 && exp_huge(yr.f))) {
                sc.fb = true;
                break;
            }
            if (yr.kind == 1 && xm.kind != APB_ZERO && xm.e + yr.f > sc.e_rad) sc.e_rad = xm.e + yr.f;
            if (xr.kind == 1 && ym.kind != APB_ZERO && ym.e + xr.f > sc.e_rad) sc.e_rad = ym.e + xr.f;
            if (xr.kind == 1 && yr.kind == 1 && xr.f + yr.f > sc.e_rad) sc.e_rad = xr.f + yr.f;
        }
    }
    return finish_plan(sc.e_max, sc.e_min, sc.e_rad, sc.nnz, sc.fb, total, p, disable_red);
}

__device__ void g_rad_term(uint64_t& srad, const GBall& x, const GBall& y, int64_t e_rad) {
    if (y.r.kind != 0 && x.m.kind != APB_ZERO)
        srad += srad_term((x.m.d[x.m.n - 1] >> 34) + 1, x.m.e, y.r.b, y.r.f, e_rad);
    if (x.r.kind != 0 && y.m.kind != APB_ZERO)
        srad += srad_term((y.m.d[y.m.n - 1] >> 34) + 1, y.m.e, x.r.b, x.r.f, e_rad);
    if (x.r.kind != 0 && y.r.kind != 0) srad += srad_term(x.r.b, x.r.f, y.r.b, y.r.f, e_rad);
}

// one dot over a term callback; writes the output ball at `ob`
template <class GetTerm>
__device__ void g_dot(GetTerm&& get, int64_t total, int64_t p, bool approx, bool disable_red,
                      const BallsOut& out, int64_t ob, apb_dot_state* st, uint64_t* accout,
                      int64_t acc_stride, int* status) {
    GBall xs, ys;
    Plan pl = g_setup(get, total, p, !approx, disable_red, xs, ys);
    if (pl.status == 2) {
        if (st) write_state(st, pl, 0, 0);
        GFloat<1> z;
        z.kind = APB_ZERO;
        z.neg = 0;
        z.e = 0;
        z.n = 0;
        gf_store(out, ob, z, mag_zero(), status);
        return;
    }
    if (pl.status == 1) {
        if (st) write_state(st, pl, 0, 0);
        // fallback_ball / fallback_approx (src/dot.cpp:325-344)
        GBall acc;
        GF tmp;
        acc.m.kind = APB_ZERO;
        acc.m.neg = 0;
        acc.m.n = 0;
        acc.m.e = 0;
        acc.r = mag_zero();
        for (int64_t i = 0; i < total; i++) {
            bool neg;
            get(i, xs, ys, neg);
            if (neg) gf_negate(ys.m);
            if (approx) {
                gf_mul_exact(tmp, xs.m, ys.m, status);
                gf_round(tmp, p, status);
                gf_add_round(acc.m, acc.m, tmp, p, status);
            } else {
                gb_addmul(acc, xs, ys, p, tmp, status);
            }
        }
        gf_store(out, ob, acc.m, approx ? mag_zero() : acc.r, status);
        return;
    }
    uint64_t s[GCAP];
    for (int j = 0; j < pl.n_s; j++) s[j] = 0;
    uint64_t err = 0, srad = 0;
    for (int64_t i = 0; i < total; i++) {
        bool neg;
        get(i, xs, ys, neg);
        if (xs.m.kind != APB_ZERO && ys.m.kind != APB_ZERO) g_acc_term(pl, s, err, xs.m, ys.m, neg);
        if (!approx) g_rad_term(srad, xs, ys, pl.e_rad);
    }
    if (st) write_state(st, pl, err, srad);
    if (accout)
        for (int j = 0; j < pl.n_s && j < acc_stride; j++) accout[j] = s[j];
    finalize_store<GCAP>(pl, s, err, srad, p, !approx, out, ob, status);
}

__global__ void __launch_bounds__(128) dot_generic_kernel(DotArgs A, int fallback_only) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= A.batch) return;
    if (fallback_only && !A.fb_flag[b]) return;
    int64_t ex0, xst, ey0, yst, nb;
    dot_extent(A, b, ex0, xst, ey0, yst, nb);
    const int64_t total = nb + (A.has_init ? 1 : 0);
    auto get = [&](int64_t i, GBall& xs, GBall& ys, bool& neg) {
        if (i < nb) {
            gb_load(xs, A.x, ex0 + i * xst);
            gb_load(ys, A.y, ey0 + i * yst);
            neg = A.subtract != 0;
        } else {
            gb_load(xs, A.init, b);
            gb_one(ys);
            neg = false;
        }
    };
    g_dot(get, total, A.prec, A.mode == APB_DOT_APPROX, A.disable_reduction != 0, A.out, b,
          A.state ? A.state + b : nullptr, A.acc ? A.acc + b * A.acc_stride : nullptr, A.acc_stride,
          A.status);
}

// ------------------------------------------------------------ wide dots
// Runtime-size operands and accumulators (p > 512 or n_s > 9, e.g. config 5's
// p = 1024 / 4096 sweep): one warp per dot, lanes striding over the terms, each
// lane with a private n_s-limb accumulator (the generic g_acc_term incl.
// mulhigh_approx, thread-local), then a warp-shuffle carry-propagating reduction
// of the 32 accumulators (two's complement addition mod 2^(64 n_s) is
// associative) and lane 0's dot_finalize.  Special-value dots are flagged for the
// thread-per-dot fallback pass (dot_generic_kernel).
__global__ void __launch_bounds__(128) dot_wide_kernel(DotArgs A) {
    const int lane = threadIdx.x & 31;
    const int64_t b = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (b >= A.batch) return;
    int64_t ex0, xst, ey0, yst, nb;
    dot_extent(A, b, ex0, xst, ey0, yst, nb);
    const int64_t total = nb + (A.has_init ? 1 : 0);
    const bool approx = A.mode == APB_DOT_APPROX;
    auto get = [&](int64_t i, GBall& xs, GBall& ys, bool& neg) {
        if (i < nb) {
            gb_load(xs, A.x, ex0 + i * xst);
            gb_load(ys, A.y, ey0 + i * yst);
            neg = A.subtract != 0;
        } else {
            gb_load(xs, A.init, b);
            gb_one(ys);
            neg = false;
        }
    };
    // ---- pass 1: setup_core over this lane's terms, warp-reduced
    GBall xs, ys;
    ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
    const bool track_min = A.prec > 128;
    for (int64_t i = lane; i < total && !sc.fb; i += 32) {
        bool neg;
        get(i, xs, ys, neg);
        const GF& xm = xs.m;
        const GF& ym = ys.m;
        if (!(xm.kind == APB_ZERO || xm.kind == APB_FINITE) || !(ym.kind == APB_ZERO || ym.kind == APB_FINITE) ||
            (xm.kind != APB_ZERO && exp_huge(xm.e)) || (ym.kind != APB_ZERO && exp_huge(ym.e))) {
            sc.fb = true;
            break;
        }
        if (xm.kind != APB_ZERO && ym.kind != APB_ZERO) {
            sc.nnz++;
            const int64_t ee = xm.e + ym.e;
            if (ee > sc.e_max) sc.e_max = ee;
            if (track_min) {
                const int64_t lo = ee - 64 * (int64_t)(xm.n + ym.n);
                if (lo < sc.e_min) sc.e_min = lo;
            }
        }
        if (!approx) {
            const Mag& xr = xs.r;
            const Mag& yr = ys.r;
            if (xr.kind == 2 || yr.kind == 2 || (xr.kind == 1 && exp_huge(xr.f)) || (yr.kind == 1 && exp_huge(yr.f))) {
                sc.fb = true;
                break;
            }
            if (yr.kind == 1 && xm.kind != APB_ZERO && xm.e + yr.f > sc.e_rad) sc.e_rad = xm.e + yr.f;
            if (xr.kind == 1 && ym.kind != APB_ZERO && ym.e + xr.f > sc.e_rad) sc.e_rad = ym.e + xr.f;
            if (xr.kind == 1 && yr.kind == 1 && xr.f + yr.f > sc.e_rad) sc.e_rad = xr.f + yr.f;
        }
    }
    const bool fb = __any_sync(0xffffffffu, sc.fb);
    const Plan pl = finish_plan(warp_max(sc.e_max), warp_min(sc.e_min), warp_max(sc.e_rad), warp_sum(sc.nnz), fb,
                                total, A.prec, A.disable_reduction != 0);
    if (pl.status != 0) {
        if (lane == 0) {
            if (A.state) write_state(A.state + b, pl, 0, 0);
            if (pl.status == 1) {
                A.fb_flag[b] = 1;
            } else {
                GFloat<1> z;
                z.kind = APB_ZERO;
                z.neg = 0;
                z.e = 0;
                z.n = 0;
                gf_store(A.out, b, z, mag_zero(), A.status);
            }
        }
        return;
    }
    // ---- pass 2: lane-private accumulators
    uint64_t s[GCAP];
    for (int j = 0; j < pl.n_s; j++) s[j] = 0;
    uint64_t err = 0, srad = 0;
    for (int64_t i = lane; i < total; i += 32) {
        bool neg;
        get(i, xs, ys, neg);
        if (xs.m.kind != APB_ZERO && ys.m.kind != APB_ZERO) g_acc_term(pl, s, err, xs.m, ys.m, neg);
        if (!approx) g_rad_term(srad, xs, ys, pl.e_rad);
    }
    // ---- warp reduction mod 2^(64 n_s)
    for (int o = 16; o; o >>= 1) {
        uint64_t c = 0;
        for (int j = 0; j < pl.n_s; j++) {
            const uint64_t v = __shfl_xor_sync(0xffffffffu, s[j], o);
            const uint64_t s1 = s[j] + v;
            const uint64_t c1 = s1 < v;
            const uint64_t s2 = s1 + c;
            s[j] = s2;
            c = c1 | (s2 < c);
        }
        err += __shfl_xor_sync(0xffffffffu, err, o);
        srad += __shfl_xor_sync(0xffffffffu, srad, o);
    }
    if (lane != 0) return;
    if (A.state) write_state(A.state + b, pl, err, srad);
    if (A.acc)
        for (int j = 0; j < pl.n_s && j < A.acc_stride; j++) A.acc[b * A.acc_stride + j] = s[j];
    finalize_store<GCAP>(pl, s, err, srad, A.prec, !approx, A.out, b, A.status);
}

// ------------------------------------------------------------ complex

struct CDotArgs {
    BallsView xre, xim, yre, yim;
    BallsOut ore, oim;
    apb_dot_index idx;
    int64_t n, batch, prec;
    int mode;
    int* status;
    unsigned long long* hits;  // dot_threeprod_hits (nullable)
    int force_threeprod;
    int64_t threeprod_cutoff;
};

// ---- exactness gate of the three-multiplication rewrite (src/dot.cpp:427-458).
// The rewrite is result-neutral by construction (both routes exact), so the
// device always evaluates the four-product form; the gate is evaluated only to
// count its hits like dot_threeprod_hits() (include/apball/dot.hpp:54).
APB_DEV int64_t gf_bottom(const GF& x) { return x.e - (64 * (int64_t)x.n - (int64_t)ctz64(x.d[0])); }

APB_DEV bool window_fits(const Plan& pl, int64_t top, int64_t bottom) {
    return top <= pl.e_s && bottom >= pl.e_s - 64 * (int64_t)pl.n_s;
}

// apfloat_add_exact (src/apfloat.cpp:272-306); false when the exact sum needs
// more than max_limbs limbs (or more than GCAP here)
__device__ bool gf_add_exact(GF& out, const GF& a, const GF& b, int max_limbs, int* status) {
    if (a.kind != APB_FINITE && a.kind != APB_ZERO) return false;
    if (b.kind != APB_FINITE && b.kind != APB_ZERO) return false;
    if (a.kind == APB_ZERO) return out = b, true;
    if (b.kind == APB_ZERO) return out = a, true;
    const int64_t e_top = (a.e > b.e ? a.e : b.e) + 1;
    const __int128 bot_a = (__int128)a.e - 64 * (int64_t)a.n, bot_b = (__int128)b.e - 64 * (int64_t)b.n;
    const __int128 span = (__int128)e_top - (bot_a < bot_b ? bot_a : bot_b);
    const __int128 k128 = (span + 63) / 64;
    if (k128 > max_limbs || k128 + 1 > GCAP) return false;
    const int k = (int)k128;
    const int64_t win_bot = checked_add(e_top, -64 * (int64_t)k, status);
    uint64_t A[GCAP], Bv[GCAP], S[GCAP];
    for (int i = 0; i <= k; i++) A[i] = Bv[i] = 0;
    // place |x| * 2^-win_bot (exact here: every bit lies inside the window)
    auto place = [&](uint64_t* dst, const GF& x) {
        const int64_t sh = x.e - 64 * (int64_t)x.n - win_bot;  // >= 0
        const int64_t wq = sh >> 6;
        const int bo = (int)(sh & 63);
        for (int i = 0; i < x.n; i++) {
            const int64_t w = wq + i;
            dst[w] |= x.d[i] << bo;
            if (bo && w + 1 <= k) dst[w + 1] |= x.d[i] >> (64 - bo);
        }
    };
    place(A, a);
    place(Bv, b);
    bool sign;
    auto sub = [&](const uint64_t* X, const uint64_t* Y) {
        uint64_t bw = 0;
        for (int i = 0; i <= k; i++) {
            const uint64_t x = X[i], y = Y[i];
            S[i] = x - y - bw;
            bw = (x < y) || (x == y && bw);
        }
    };
    if (a.neg == b.neg) {
        uint64_t c = 0;
        for (int i = 0; i <= k; i++) {
            const uint64_t s1 = A[i] + Bv[i];
            const uint64_t c1 = s1 < A[i];
            const uint64_t s2 = s1 + c;
            c = c1 | (s2 < s1);
            S[i] = s2;
        }
        sign = a.neg;
    } else {
        int cmp = 0;
        for (int i = k; i >= 0 && !cmp; i--) cmp = A[i] > Bv[i] ? 1 : (A[i] < Bv[i] ? -1 : 0);
        if (cmp >= 0) {
            sub(A, Bv);
            sign = a.neg;
        } else {
            sub(Bv, A);
            sign = b.neg;
        }
    }
    gf_normalize(out, sign ? 1 : 0, checked_add(win_bot, 64 * (int64_t)(k + 1), status), S, k + 1, status);
    return true;
}

__device__ bool threeprod_gate(const Plan& pre, const Plan& pim, const GF& a, const GF& b, const GF& c,
                               const GF& d, bool force, int64_t cutoff, int* status) {
    if (a.kind == APB_ZERO || b.kind == APB_ZERO || c.kind == APB_ZERO || d.kind == APB_ZERO) return false;
    if (!force) {
        if ((a.n < b.n ? a.n : b.n) < cutoff) return false;
        if ((c.n < d.n ? c.n : d.n) < cutoff) return false;
    }
    const int64_t ba = gf_bottom(a), bb = gf_bottom(b), bc = gf_bottom(c), bd = gf_bottom(d);
    // four-route products stay inside their windows; rewrite terms likewise
    if (!window_fits(pre, a.e + c.e, ba + bc)) return false;
    if (!window_fits(pre, b.e + d.e, bb + bd)) return false;
    if (!window_fits(pim, a.e + d.e, ba + bd)) return false;
    if (!window_fits(pim, b.e + c.e, bb + bc)) return false;
    if (!window_fits(pim, a.e + c.e, ba + bc)) return false;
    if (!window_fits(pim, b.e + d.e, bb + bd)) return false;
    const int cap = a.n + b.n + c.n + d.n + 8;
    GF sab, scd;
    if (!gf_add_exact(sab, a, b, cap, status)) return false;
    if (!gf_add_exact(scd, c, d, cap, status)) return false;
    if (sab.kind == APB_ZERO || scd.kind == APB_ZERO) return true;  // e = 0 fits trivially
    // e = (a+b)(c+d): bottom = sum of bottoms exactly; top is e_ab + e_cd or one less
    const int64_t ebot = gf_bottom(sab) + gf_bottom(scd);
    if (sab.n + scd.n <= GCAP) {
        GF e;
        gf_mul_exact(e, sab, scd, status);
        return window_fits(pim, e.e, gf_bottom(e));
    }
    const int64_t etop_hi = sab.e + scd.e;
    if (window_fits(pim, etop_hi, ebot)) return true;
    return false;  // (only the exact top could still fit: conservatively counted as a miss)
}

__global__ void __launch_bounds__(128) dot_complex_generic_kernel(CDotArgs A) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= A.batch) return;
    const bool approx = A.mode == APB_DOT_APPROX;
    // ComplexPartView (src/dot.cpp:52-68): re terms (a,c,+),(b,d,-); im (a,d,+),(b,c,+)
    auto get_re = [&](int64_t i, GBall& xs, GBall& ys, bool& neg) {
        int64_t j = i >> 1;
        int64_t ex = x_elem(A.idx, b, j), ey = y_elem(A.idx, b, j);
        if (i & 1) {
            gb_load(xs, A.xim, ex);
            gb_load(ys, A.yim, ey);
            neg = true;
        } else {
            gb_load(xs, A.xre, ex);
            gb_load(ys, A.yre, ey);
            neg = false;
        }
    };
    auto get_im = [&](int64_t i, GBall& xs, GBall& ys, bool& neg) {
        int64_t j = i >> 1;
        int64_t ex = x_elem(A.idx, b, j), ey = y_elem(A.idx, b, j);
        if (i & 1) {
            gb_load(xs, A.xim, ex);
            gb_load(ys, A.yre, ey);
        } else {
            gb_load(xs, A.xre, ex);
            gb_load(ys, A.yim, ey);
        }
        neg = false;
    };
    GBall xs, ys;
    Plan pre = g_setup(get_re, 2 * A.n, A.prec, !approx, false, xs, ys);
    Plan pim = g_setup(get_im, 2 * A.n, A.prec, !approx, false, xs, ys);
    if (pre.status == 1 || pim.status == 1) {
        // complex_fallback_ball (src/dot.cpp:532-545)
        GBall are, aim;
        GF tmp;
        are.m.kind = aim.m.kind = APB_ZERO;
        are.m.neg = aim.m.neg = 0;
        are.m.n = aim.m.n = 0;
        are.m.e = aim.m.e = 0;
        are.r = aim.r = mag_zero();
        for (int64_t j = 0; j < A.n; j++) {
            bool neg;
            get_re(2 * j, xs, ys, neg);
            gb_addmul(are, xs, ys, A.prec, tmp, A.status);
            get_re(2 * j + 1, xs, ys, neg);
            gf_negate(ys.m);
            gb_addmul(are, xs, ys, A.prec, tmp, A.status);
            get_im(2 * j, xs, ys, neg);
            gb_addmul(aim, xs, ys, A.prec, tmp, A.status);
            get_im(2 * j + 1, xs, ys, neg);
            gb_addmul(aim, xs, ys, A.prec, tmp, A.status);
        }
        gf_store(A.ore, b, are.m, approx ? mag_zero() : are.r, A.status);
        gf_store(A.oim, b, aim.m, approx ? mag_zero() : aim.r, A.status);
        return;
    }
    if (A.hits && pre.status == 0 && pim.status == 0) {  // complex_core's try_rewrite (src/dot.cpp:489-501)
        unsigned long long h = 0;
        GBall ga, gbb, gc, gd;
        for (int64_t j = 0; j < A.n; j++) {
            const int64_t ex = x_elem(A.idx, b, j), ey = y_elem(A.idx, b, j);
            gb_load(ga, A.xre, ex);
            gb_load(gbb, A.xim, ex);
            gb_load(gc, A.yre, ey);
            gb_load(gd, A.yim, ey);
            if (threeprod_gate(pre, pim, ga.m, gbb.m, gc.m, gd.m, A.force_threeprod != 0, A.threeprod_cutoff,
                               A.status))
                h++;
        }
        if (h) atomicAdd(A.hits, h);
    }
    g_dot(get_re, 2 * A.n, A.prec, approx, false, A.ore, b, nullptr, nullptr, 0, A.status);
    g_dot(get_im, 2 * A.n, A.prec, approx, false, A.oim, b, nullptr, nullptr, 0, A.status);
}

// ------------------------------------------------------------ launchers

template <int L, int NS, int TPL>
static void launch_small(const DotArgs& A, cudaStream_t st) {
    const int warps = 4;  // each warp: A.dpw consecutive dots
    const int64_t nwarps = (A.batch + A.dpw - 1) / A.dpw;
    dim3 grid((unsigned)((nwarps + warps - 1) / warps));
    dot_small_kernel<L, NS, TPL><<<grid, 32 * warps, 0, st>>>(A);
    count_launch();
}

// the smallest accumulator width covering every plan for (prec, total)
static int ns_bound(int64_t prec, int64_t total) {
    auto bc = [](uint64_t v) {
        int r = 0;
        while (v) {
            r++;
            v >>= 1;
        }
        return r;
    };
    int64_t ns = (prec + (bc((uint64_t)total) + 1) + (4 + bc((uint64_t)total)) + 63) / 64;
    return (int)(ns < 2 ? 2 : ns);
}

static bool staged_ok(const DotArgs& A) {
    if (A.palen > 0) return false;  // fixed-length affine indexing only
    auto al = [](const void* p, size_t a) { return ((uintptr_t)p % a) == 0; };
    bool ok = al(A.x.mant, 8) && al(A.x.exp, 8) && al(A.x.rad_exp, 8) && al(A.x.rad_man, 4) &&
              al(A.y.mant, 8) && al(A.y.exp, 8) && al(A.y.rad_exp, 8) && al(A.y.rad_man, 4);
    if (A.has_init)
        ok = ok && al(A.init.mant, 8) && al(A.init.exp, 8) && al(A.init.rad_exp, 8) && al(A.init.rad_man, 4);
    return ok;
}

template <int L, int NS>
static void launch_staged(const DotArgs& A, cudaStream_t st) {
    const int warps = 4;
    const size_t shm = (size_t)warps * 2 * sizeof(StageBuf<L>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(dot_staged_kernel<L, NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
        attr = true;
    }
    const int64_t nwarps = (A.batch + 31) / 32;
    dim3 grid((unsigned)((nwarps + warps - 1) / warps));
    dot_staged_kernel<L, NS><<<grid, 32 * warps, shm, st>>>(A);
    count_launch();
}

// TPD lanes per dot: about 16-32 terms per lane (APB_DOT_TPD overrides; 32 = dot_small)
static int pick_tpd(int64_t total) {
    static const int env = std::getenv("APB_DOT_TPD") ? std::atoi(std::getenv("APB_DOT_TPD")) : 0;
    if (env == 1 || env == 2 || env == 4 || env == 8 || env == 16 || env == 32) return env;
    if (total <= 24) return 1;
    if (total <= 48) return 2;
    if (total <= 160) return 4;
    if (total <= 320) return 8;
    if (total <= 640) return 16;
    return 32;
}

template <int L, int NS, int TPD>
static void launch_grp(DotArgs A, cudaStream_t st) {
    constexpr int DPR = 32 / TPD;
    // rounds per warp: enough warps for >= 32 per SM, at most TPD rounds (32 dots)
    int64_t rounds = A.batch / ((int64_t)DPR * 148 * 32);
    static const int env_rounds = std::getenv("APB_DOT_ROUNDS") ? std::atoi(std::getenv("APB_DOT_ROUNDS")) : 0;
    if (env_rounds > 0) rounds = env_rounds;  // tuning hook
    rounds = rounds < 1 ? 1 : (rounds > TPD ? TPD : rounds);
    A.dpw = (int)(DPR * rounds);
    const int warps = 4;
    const int64_t nwarps = (A.batch + A.dpw - 1) / A.dpw;
    dim3 grid((unsigned)((nwarps + warps - 1) / warps));
    dot_grp_kernel<L, NS, TPD><<<grid, 32 * warps, 0, st>>>(A);
    count_launch();
}

template <int TPD, int RS, bool UNIT, bool PF>
static void launch_reg_u(const DotArgs& A, cudaStream_t st) {
    constexpr int DPR = 32 / TPD;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dot_reg_kernel<TPD, RS, UNIT, PF>, 128, 0);
        if (occ < 1) occ = 1;
    }
    const int64_t ngroups = (A.batch + DPR - 1) / DPR;
    const int64_t blocks = std::min<int64_t>((ngroups + 3) / 4, (int64_t)148 * occ);
    dot_reg_kernel<TPD, RS, UNIT, PF><<<(unsigned)blocks, 128, 0, st>>>(A, ngroups);
    count_launch();
}
template <int TPD, int RS>
static void launch_reg(const DotArgs& A, cudaStream_t st) {
    // L2 prefetch of the next group: opt-in (APB_REG_PF=1), measured slower on config 1
    static const bool pf = std::getenv("APB_REG_PF") != nullptr;
    const bool unit = A.idx.xstep == 1 && A.idx.ystep == 1;
    const bool flat = unit && A.idx.bdiv == 1 && A.idx.xs1 == A.n && A.idx.ys1 == A.n && pf;
    if (flat)
        launch_reg_u<TPD, RS, true, true>(A, st);
    else if (unit)
        launch_reg_u<TPD, RS, true, false>(A, st);
    else
        launch_reg_u<TPD, RS, false, false>(A, st);
}

// register-resident kernel (dot_reg.cuh): <= 2-limb operands, n_s <= 3, no initial
// value, 33 <= n <= 128 terms (RS = ceil(n / 32) slots); APB_DOT_NOREG=1 keeps the
// lane-group / warp kernels
static bool try_reg(const DotArgs& A, int Lin, int nsb, int64_t total, cudaStream_t st) {
    static const bool off = std::getenv("APB_DOT_NOREG") != nullptr;
    static const int env_tpd = std::getenv("APB_REG_TPD") ? std::atoi(std::getenv("APB_REG_TPD")) : 0;
    if (off || Lin > 2 || nsb > 3 || A.has_init || A.palen > 0 || total > 128 || total <= 32) return false;
    if (env_tpd == 16 && total > 96 && total <= 112) {
        launch_reg<16, 7>(A, st);
        return true;
    }
    if (total > 96) launch_reg<32, 4>(A, st);
    else if (total > 64) launch_reg<32, 3>(A, st);
    else launch_reg<32, 2>(A, st);
    return true;
}

template <int L, int NS>
static bool try_small_tpl(const DotArgs& A, int64_t total, cudaStream_t st) {
    if (L == 2 && A.batch >= 148 * BLK_DOTS * 4 && blk_ok(A, L)) {  // contiguous batch: bulk-staged
        launch_blk<L, NS>(A, st);
        return true;
    }
    const int tpd = pick_tpd(total);
    if (tpd < 32 && !std::getenv("APB_DOT_KEEP") && !std::getenv("APB_DOT_STAGE")) {
        switch (tpd) {
            case 1: launch_grp<L, NS, 1>(A, st); return true;
            case 2: launch_grp<L, NS, 2>(A, st); return true;
            case 4: launch_grp<L, NS, 4>(A, st); return true;
            case 8: launch_grp<L, NS, 8>(A, st); return true;
            default: launch_grp<L, NS, 16>(A, st); return true;
        }
    }
    // Default: one warp per 32 dots, operands re-read from L1/L2 per term
    // (measured fastest on config 1: 0.38 ms vs 0.53 ms register-resident and
    // 0.60 ms cp.async-staged).  The other two variants stay reachable for
    // tuning and are covered by the GPU tests through these hooks.
    static const bool keep = std::getenv("APB_DOT_KEEP") != nullptr;
    static const bool stage = std::getenv("APB_DOT_STAGE") != nullptr;
    if (total <= STG_T && L <= 2 && stage && staged_ok(A)) {
        launch_staged<L, NS>(A, st);
    } else if (total <= 32 * 4 && L <= 2 && keep) {
        launch_small<L, NS, 4>(A, st);
    } else {
        launch_small<L, NS, 0>(A, st);
    }
    return true;
}

int dot_dispatch(DotArgs& A, int Lin, int64_t total, cudaStream_t st);

int dot_batch_launch(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                     int subtract, const apb_dot_index* idx, int64_t n, int64_t batch, int64_t prec,
                     int mode, const apb_dot_tuning* tuning, apb_balls* out, apb_dot_state* state,
                     uint64_t* acc, int64_t acc_stride, cudaStream_t st) {
    if (batch == 0) return APB_OK;
    DotArgs A;
    A.x = view_of(x);
    A.y = view_of(y);
    A.has_init = initial != nullptr;
    A.init = initial ? view_of(initial) : view_of(x);
    A.out = out_of(out);
    A.idx = *idx;
    A.n = n;
    A.batch = batch;
    A.prec = prec;
    A.mode = mode;
    A.subtract = subtract;
    A.disable_reduction = tuning ? tuning->disable_precision_reduction : 0;
    A.state = state;
    A.acc = acc;
    A.acc_stride = acc_stride;
    const int64_t total = n + (initial ? 1 : 0);
    int Lin = x->L > y->L ? x->L : y->L;
    if (initial && initial->L > Lin) Lin = initial->L;
    return dot_dispatch(A, Lin, total, st);
}

// template dispatch + fallback pass for a prepared DotArgs (total = max terms per dot)
int dot_dispatch(DotArgs& A, int Lin, int64_t total, cudaStream_t st) {
    const int64_t batch = A.batch, prec = A.prec;
    Workspace& ws = workspace();
    A.status = ws.status_dev;
    A.fb_flag = (uint8_t*)ws.scratch(st, (size_t)batch, 20);
    if (!A.fb_flag) {
        set_error("out of device memory (dot flags)");
        return APB_ERR_CUDA;
    }
    cudaMemsetAsync(A.fb_flag, 0, (size_t)batch, st);
    // 32 dots per warp once the batch fills >= 8 warps per SM that way; fewer
    // (down to one) for small batches so every SM gets warps
    A.dpw = batch >= (int64_t)32 * 148 * 8 ? 32 : (int)std::max<int64_t>(1, batch / (148 * 8));
    const int nsb = ns_bound(prec, total);
    A.mant16 = A.x.L == 2 && A.y.L == 2 && ((uintptr_t)A.x.mant % 16) == 0 && ((uintptr_t)A.y.mant % 16) == 0;
    const int tok = prof_begin("dot", st);
    bool small = true;
    if (try_reg(A, Lin, nsb, total, st)) {
    } else if (Lin <= 1 && nsb <= 3) try_small_tpl<1, 3>(A, total, st);
    else if (Lin <= 2 && nsb <= 3) try_small_tpl<2, 3>(A, total, st);
    else if (Lin <= 2 && nsb <= 5) try_small_tpl<2, 5>(A, total, st);
    else if (Lin <= 4 && nsb <= 5) try_small_tpl<4, 5>(A, total, st);
    else if (Lin <= 4 && nsb <= 9) try_small_tpl<4, 9>(A, total, st);
    else if (Lin <= 8 && nsb <= 9) try_small_tpl<8, 9>(A, total, st);
    else small = false;
    // wide precisions: warp per dot (APB_DOT_GENERIC=1: the thread-per-dot kernel alone)
    static const bool generic_only = std::getenv("APB_DOT_GENERIC") != nullptr;
    bool flagged = small;
    if (!small && !generic_only) {
        dot_wide_kernel<<<(unsigned)((batch * 32 + 127) / 128), 128, 0, st>>>(A);
        count_launch();
        flagged = true;
    }
    const unsigned gthreads = 128;
    dim3 ggrid((unsigned)((batch + gthreads - 1) / gthreads));
    dot_generic_kernel<<<ggrid, gthreads, 0, st>>>(A, flagged ? 1 : 0);
    prof_end(tok, st);
    count_launch();
    return APB_OK;
}

// ------------------------------------------------------------ poly (§8(f) row 2)

// poly_mullow_classical (src/poly.cpp:11-26): output k is one dot over
// (a_i, b_{k-i}), i in [max(0, k+1-|b|), min(k, |a|-1)], with a negative step on
// b; all len outputs are one batch of variable-length dots.
int poly_mullow_launch(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                       int64_t prec, apb_balls* out, cudaStream_t st) {
    if (len == 0) return APB_OK;
    DotArgs A;
    A.x = view_of(a);
    A.y = view_of(b);
    A.has_init = false;
    A.init = view_of(a);
    A.out = out_of(out);
    std::memset(&A.idx, 0, sizeof A.idx);
    A.idx.bdiv = 1;
    A.palen = alen;
    A.pblen = blen;
    const int64_t nmax = alen < blen ? alen : blen;
    A.n = nmax;
    A.batch = len;
    A.prec = prec;
    A.mode = APB_DOT_BALL;
    A.subtract = 0;
    A.disable_reduction = 0;
    A.state = nullptr;
    A.acc = nullptr;
    A.acc_stride = 0;
    if (alen == 0 || blen == 0) A.palen = -1;  // every output is the exact zero
    if (A.palen < 0) {
        A.palen = 1;
        A.pblen = 0;  // n = 0 for every k
    }
    return dot_dispatch(A, a->L > b->L ? a->L : b->L, nmax > 0 ? nmax : 1, st);
}

// apfloat_mul_u64_exact (src/apfloat.cpp:178-186)
__device__ void gf_mul_u64_exact(GF& out, const GF& x, uint64_t k, int* status) {
    if (x.kind != APB_FINITE) {
        out = x;
        if (k == 0 && (x.kind == APB_PINF || x.kind == APB_NINF)) out.kind = APB_NAN;
        return;
    }
    if (k == 0) {
        out.kind = APB_ZERO;
        out.neg = 0;
        out.e = 0;
        out.n = 0;
        return;
    }
    uint64_t prod[GCAP];
    uint64_t cy = 0;
    for (int i = 0; i < x.n; i++) {
        const unsigned __int128 t = (unsigned __int128)x.d[i] * k + cy;
        prod[i] = (uint64_t)t;
        cy = (uint64_t)(t >> 64);
    }
    prod[x.n] = cy;
    gf_normalize(out, x.neg, checked_add(x.e, 64, status), prod, x.n + 1, status);
}

// mag_inv_u64_upper (src/mag.cpp:155-164)
APB_DEV Mag mag_inv_u64(uint64_t k) {
    const unsigned len = bitw64(k);
    if ((k & (k - 1)) == 0) return mag_parts(kMagOne >> 1, 2 - (int64_t)len);
    const unsigned __int128 num = (unsigned __int128)1 << (30 - 1 + len);
    uint64_t q = (uint64_t)(num / k);
    if (num % k) q++;
    return mag_parts(q, 1 - (int64_t)len);
}

// ball_div_u64 (src/ball.cpp:38-43) with apfloat_div_u64 (src/apfloat.cpp:308-331)
__device__ void gb_div_u64(GBall& out, const GBall& x, uint64_t k, int64_t p, int* status) {
    if (x.m.kind == APB_NAN) {
        out.m.kind = APB_NAN;
        out.m.neg = 0;
        out.m.e = 0;
        out.m.n = 0;
        out.r = mag_inf();
        return;
    }
    p = p < 2 ? 2 : p;
    Mag err = mag_zero();
    if (x.m.kind != APB_FINITE) {
        out.m = x.m;
    } else {
        const int n = x.m.n;
        const int64_t wl = (int64_t)n > p / 64 + 1 ? n : p / 64 + 1;
        const int w = (int)wl + 1;
        uint64_t q[GCAP];
        uint64_t rem = 0;
        for (int i = w - 1; i >= 0; i--) {
            const uint64_t num = i + n >= w ? x.m.d[i + n - w] : 0ull;
            const unsigned __int128 cur = ((unsigned __int128)rem << 64) | num;
            q[i] = (uint64_t)(cur / k);
            rem = (uint64_t)(cur % k);
        }
        gf_normalize(out.m, x.m.neg, x.m.e, q, w, status);
        err = gf_round(out.m, p, status);
        if (rem) err = mag_add(err, mag_from_u64(1, checked_add(x.m.e, -64 * (int64_t)w, status)));
    }
    out.r = mag_add(err, mag_mul(x.r, mag_inv_u64(k)));
}

// series_exp_basecase (src/poly.cpp:28-46): b_0 = 1, b_k = (sum_j (j a_j) b_{k-j}) / k.
// The recurrence is sequential; one thread walks it with the generic fused dot
// (the same Algorithm 1 restatement as dot_generic_kernel), reading b from the
// output as it is produced.  ja (j a_j, exact) is staged in `ja` (L_a + 1 limbs).
// one dot (Algorithm 1 over a term callback) computed by a whole warp: lanes
// stride over the terms with private runtime-size accumulators, shuffle carry
// reduction, lane 0 finalizes into (out, ob); special values: lane 0 runs the
// fallback (ball_fallback_addmul per term) exactly as g_dot does
template <class GetTerm>
__device__ void warp_g_dot(GetTerm&& get, int64_t total, int64_t p, const BallsOut& out, int64_t ob, int* status) {
    const int lane = threadIdx.x & 31;
    GBall xs, ys;
    ScanAcc sc{INT64_MIN, INT64_MAX, INT64_MIN, 0, false};
    const bool track_min = p > 128;
    for (int64_t i = lane; i < total && !sc.fb; i += 32) {
        bool neg;
        get(i, xs, ys, neg);
        const GF& xm = xs.m;
        const GF& ym = ys.m;
        if (!(xm.kind == APB_ZERO || xm.kind == APB_FINITE) || !(ym.kind == APB_ZERO || ym.kind == APB_FINITE) ||
            (xm.kind != APB_ZERO && exp_huge(xm.e)) || (ym.kind != APB_ZERO && exp_huge(ym.e))) {
            sc.fb = true;
            break;
        }
        if (xm.kind != APB_ZERO && ym.kind != APB_ZERO) {
            sc.nnz++;
            const int64_t ee = xm.e + ym.e;
            if (ee > sc.e_max) sc.e_max = ee;
            if (track_min) {
                const int64_t lo = ee - 64 * (int64_t)(xm.n + ym.n);
                if (lo < sc.e_min) sc.e_min = lo;
            }
        }
        const Mag& xr = xs.r;
        const Mag& yr = ys.r;
        if (xr.kind == 2 || yr.kind == 2 || (xr.kind == 1 && exp_huge(xr.f)) || (yr.kind == 1 && exp_huge(yr.f))) {
            sc.fb = true;
            break;
        }
        if (yr.kind == 1 && xm.kind != APB_ZERO && xm.e + yr.f > sc.e_rad) sc.e_rad = xm.e + yr.f;
        if (xr.kind == 1 && ym.kind != APB_ZERO && ym.e + xr.f > sc.e_rad) sc.e_rad = ym.e + xr.f;
        if (xr.kind == 1 && yr.kind == 1 && xr.f + yr.f > sc.e_rad) sc.e_rad = xr.f + yr.f;
    }
    const bool fb = __any_sync(0xffffffffu, sc.fb);
    const Plan pl = finish_plan(warp_max(sc.e_max), warp_min(sc.e_min), warp_max(sc.e_rad), warp_sum(sc.nnz), fb,
                                total, p, false);
    if (pl.status != 0) {
        if (lane == 0) g_dot(get, total, p, false, false, out, ob, nullptr, nullptr, 0, status);  // zero / fallback
        return;
    }
    uint64_t s[GCAP];
    for (int j = 0; j < pl.n_s; j++) s[j] = 0;
    uint64_t err = 0, srad = 0;
    for (int64_t i = lane; i < total; i += 32) {
        bool neg;
        get(i, xs, ys, neg);
        if (xs.m.kind != APB_ZERO && ys.m.kind != APB_ZERO) g_acc_term(pl, s, err, xs.m, ys.m, neg);
        g_rad_term(srad, xs, ys, pl.e_rad);
    }
    for (int o = 16; o; o >>= 1) {
        uint64_t c = 0;
        for (int j = 0; j < pl.n_s; j++) {
            const uint64_t v = __shfl_xor_sync(0xffffffffu, s[j], o);
            const uint64_t s1 = s[j] + v;
            const uint64_t c1 = s1 < v;
            const uint64_t s2 = s1 + c;
            s[j] = s2;
            c = c1 | (s2 < c);
        }
        err += __shfl_xor_sync(0xffffffffu, err, o);
        srad += __shfl_xor_sync(0xffffffffu, srad, o);
    }
    if (lane == 0) finalize_store<GCAP>(pl, s, err, srad, p, true, out, ob, status);
}

// series_exp_basecase (src/poly.cpp:29-46) on one warp: b_0 = 1, then for
// k = 1.. the dot sum_{i<k} (i+1) a_{i+1} b_{k-1-i} (one warp-wide dot, lanes
// over the terms) and lane 0's b_k = dot / k (ball_div_u64); the recurrence
// itself is sequential.  (APB_SERIES_SERIAL=1: the previous one-thread version.)
__global__ void series_exp_kernel(BallsView a, int64_t alen, int64_t len, int64_t prec, BallsOut out,
                                  BallsOut ja, BallsOut sdot, int* status, int serial) {
    if (blockIdx.x != 0) return;
    const int lane = threadIdx.x & 31;
    if (threadIdx.x >= 32) return;
    GBall x, y, t;
    // ja[j] = (j a_j exact, mag_mul_up(rad, Mag::from_u64_upper(j))), zero beyond |a|
    for (int64_t j = lane; j < len; j += 32) {
        if (j >= 1 && j < alen) {
            gb_load(x, a, j);
            gf_mul_u64_exact(t.m, x.m, (uint64_t)j, status);
            t.r = mag_mul(x.r, mag_from_u64((uint64_t)j, 0));
        } else {
            t.m.kind = APB_ZERO;
            t.m.neg = 0;
            t.m.e = 0;
            t.m.n = 0;
            t.r = mag_zero();
        }
        gf_store(ja, j, t.m, t.r, status);
    }
    if (lane == 0) {  // b_0 = Ball::from_i64(1)
        GFloat<1> one;
        one.kind = APB_FINITE;
        one.neg = 0;
        one.e = 1;
        one.n = 1;
        one.d[0] = 1ull << 63;
        gf_store(out, 0, one, mag_zero(), status);
    }
    __syncwarp();
    const BallsView jav{ja.mant, ja.exp, ja.kind, ja.rad_man, ja.rad_exp, ja.L};
    const BallsView bv{out.mant, out.exp, out.kind, out.rad_man, out.rad_exp, out.L};
    const BallsView sv{sdot.mant, sdot.exp, sdot.kind, sdot.rad_man, sdot.rad_exp, sdot.L};
    for (int64_t k = 1; k < len; k++) {
        auto get = [&](int64_t i, GBall& xs, GBall& ys, bool& neg) {
            gb_load(xs, jav, 1 + i);
            gb_load(ys, bv, k - 1 - i);
            neg = false;
        };
        if (serial) {
            if (lane == 0) g_dot(get, k, prec, false, false, sdot, 0, nullptr, nullptr, 0, status);
        } else {
            warp_g_dot(get, k, prec, sdot, 0, status);
        }
        if (lane == 0) {
            gb_load(x, sv, 0);
            gb_div_u64(t, x, (uint64_t)k, prec, status);
            gf_store(out, k, t.m, t.r, status);
        }
        __syncwarp();  // b_k (global, written by lane 0) is read by every lane next step
    }
}

int series_exp_launch(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out,
                      cudaStream_t st) {
    if (len == 0) return APB_OK;
    Workspace& ws = workspace();
    const int La = a->L + 1, Ls = out->L;
    const size_t cnt = (size_t)len;
    // ja (La limbs) and the dot scratch (one ball) in workspace slots 21-29
    apb_balls ja{(uint64_t*)ws.scratch(st, cnt * La * 8, 21), (int64_t*)ws.scratch(st, cnt * 8, 22),
                 (uint8_t*)ws.scratch(st, cnt, 23), (uint32_t*)ws.scratch(st, cnt * 4, 24),
                 (int64_t*)ws.scratch(st, cnt * 8, 25), (int64_t)len, La};
    apb_balls sd{(uint64_t*)ws.scratch(st, (size_t)Ls * 8, 26), (int64_t*)ws.scratch(st, 8, 27),
                 (uint8_t*)ws.scratch(st, 1, 28), (uint32_t*)ws.scratch(st, 4, 29),
                 (int64_t*)ws.scratch(st, 8, 30), 1, Ls};
    if (!ja.mant || !ja.exp || !ja.kind || !ja.rad_man || !ja.rad_exp || !sd.mant || !sd.exp || !sd.kind ||
        !sd.rad_man || !sd.rad_exp) {
        set_error("out of device memory (series scratch)");
        return APB_ERR_CUDA;
    }
    static const int serial = std::getenv("APB_SERIES_SERIAL") ? 1 : 0;  // test hook
    series_exp_kernel<<<1, 32, 0, st>>>(view_of(a), alen, len, prec, out_of(out), out_of(&ja), out_of(&sd),
                                        ws.status_dev, serial);
    count_launch();
    return cuda_check(cudaGetLastError(), "series_exp");
}

int dot_complex_launch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                       const apb_balls* yim, const apb_dot_index* idx, int64_t n, int64_t batch,
                       int64_t prec, int mode, apb_balls* ore, apb_balls* oim, cudaStream_t st,
                       const apb_dot_tuning* tuning, uint64_t* hits) {
    if (batch == 0) return APB_OK;
    CDotArgs A;
    A.xre = view_of(xre);
    A.xim = view_of(xim);
    A.yre = view_of(yre);
    A.yim = view_of(yim);
    A.ore = out_of(ore);
    A.oim = out_of(oim);
    A.idx = *idx;
    A.n = n;
    A.batch = batch;
    A.prec = prec;
    A.mode = mode;
    A.status = workspace().status_dev;
    A.hits = (unsigned long long*)hits;
    A.force_threeprod = tuning ? tuning->force_threeprod : 0;
    A.threeprod_cutoff = tuning && tuning->threeprod_cutoff_limbs > 0 ? tuning->threeprod_cutoff_limbs : 128;
    const unsigned t = 128;
    dot_complex_generic_kernel<<<(unsigned)((batch + t - 1) / t), t, 0, st>>>(A);
    count_launch();
    return APB_OK;
}

}  // namespace apb
