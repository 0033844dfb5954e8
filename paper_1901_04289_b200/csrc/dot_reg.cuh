// dot_reg.cuh - register-resident dot kernel for config-1-shaped batches
// (included by dot_kernels.cu; shares DotArgs / Plan / finish_plan /
// finalize_store with the other dot kernels).
//
// Eligible batches: both operands of <= 2 limbs, every plan's accumulator
// window n_s <= 3 (ns_bound), n <= TPD * RS terms per dot, no initial value.
// TPD lanes own one dot and RS register slots each: every term of the dot is
// loaded ONCE (one coalesced pass over the five SoA arrays of x and y) and both
// passes of Algorithm 1 -- the setup scan (setup_core, src/dot.cpp:72-134) and
// the accumulation (dot_accumulate_term + radius_pass_term, src/dot.cpp:229-273,
// 346-358) -- read registers.  The dot kernels of round 1 re-read the operands
// for the second pass and did the term arithmetic on 64-bit limbs with generic
// barrel shifts (~560 instructions per term on config 1); here a term is:
//
//   * the 4x4 32-bit-limb product P = x * y of the top-aligned mantissas (PTX
//     mad.lo/hi carry chains);
//   * its placement floor(P / 2^r), r = shift + 256 - 64 n_s: because every
//     term's shift is >= extend (e_s = e_max + extend) the limb offset q = r/32 is
//     at least q0 = 8 - 2 n_s, so terms within 2^-(64 - extend) of the largest
//     take a two-way limb select (q in {q0, q0+1}) plus 2 n_s funnel shifts; the
//     others (far smaller terms) a generic select;
//   * err += 1 iff the floor dropped nonzero bits (the limbs below q and the low
//     t = r mod 32 bits of limb q) -- exactly the strip / drop rule of
//     accumulate_aligned (src/dot.cpp:139-173);
//   * the two's complement add/subtract of the 6-limb contribution as one
//     carry chain: acc += (C xor m) + neg, m = -neg.
//
// Two's complement addition modulo 2^192 is associative, so the lane
// accumulators combine by a shuffle carry chain and the result equals the
// reference's sequential sum bit for bit (for n_s = 2 the low 128 bits are the
// sum modulo 2^128).  Finalize (dot_finalize, src/dot.cpp:306-321) runs on
// parked states, one dot per lane, as in dot_grp_kernel.
#pragma once
// (included inside namespace apb)

// Exponents: the five SoA exponent fields are int64 (ApFloat / Mag exponents);
// every exponent of a dot that takes this kernel lies in [-2^29, 2^29) (checked
// per term, unconditionally), so all exponent sums, the plan and the radius
// shifts are 32-bit.  A dot with a larger exponent, a special value (inf / nan,
// infinite radius) is flagged for dot_generic_kernel, which recomputes it from
// scratch (the same Algorithm 1 restatement incl. the Fallback semantics).

struct RTerm {
    uint32_t X[4], Y[4];  // top-aligned mantissas as 32-bit limbs (L = 2 view)
    int32_t ee;           // ex + ey
    int32_t s1, s2, s3;   // ex + fy, ey + fx, fx + fy (radius exponent sums)
    uint32_t rx, ry;      // radius mantissas (0 = exact)
    uint32_t k;           // kx | ky << 8; 0 for an empty slot
};

APB_DEV void split64(uint64_t v, uint32_t& lo, uint32_t& hi) {
    lo = (uint32_t)v;
    hi = (uint32_t)(v >> 32);
}

// nonzero unless v in [-2^29, 2^29)
APB_DEV uint32_t exp_out(int64_t v) {
    const int32_t lo = (int32_t)v, hi = (int32_t)(v >> 32);
    const int32_t a = lo >> 29;
    return (uint32_t)((hi ^ a) | (a ^ (a >> 2)));
}

// per-dot lane pointers into the SoA arrays (element ex0 + sub * xstep)
struct RPtrs {
    const uint8_t *kx, *ky;
    const int64_t *ex, *ey, *fx, *fy;
    const uint32_t *rx, *ry;
    const uint64_t *mx, *my;
};

// term `off` elements past the lane's first element; operands with L <= 2.
// bad |= exponent-range violations (dot goes to the generic kernel).
APB_DEV void reg_load(RTerm& t, const DotArgs& A, const RPtrs& q, int64_t offx, int64_t offy, bool with_radius,
                      uint32_t& bad) {
    const uint32_t kx = __ldg(q.kx + offx), ky = __ldg(q.ky + offy);
    const int64_t px = __ldg(q.ex + offx), py = __ldg(q.ey + offy);
    uint64_t xm0, xm1, ym0, ym1;
    if (A.mant16) {
        const ulonglong2 vx = __ldg(reinterpret_cast<const ulonglong2*>(q.mx) + offx);
        const ulonglong2 vy = __ldg(reinterpret_cast<const ulonglong2*>(q.my) + offy);
        xm0 = vx.x;
        xm1 = vx.y;
        ym0 = vy.x;
        ym1 = vy.y;
    } else {
        if (A.x.L == 2) {
            xm0 = __ldg(q.mx + 2 * offx);
            xm1 = __ldg(q.mx + 2 * offx + 1);
        } else {
            xm0 = 0;
            xm1 = __ldg(q.mx + offx);
        }
        if (A.y.L == 2) {
            ym0 = __ldg(q.my + 2 * offy);
            ym1 = __ldg(q.my + 2 * offy + 1);
        } else {
            ym0 = 0;
            ym1 = __ldg(q.my + offy);
        }
    }
    split64(xm0, t.X[0], t.X[1]);
    split64(xm1, t.X[2], t.X[3]);
    split64(ym0, t.Y[0], t.Y[1]);
    split64(ym1, t.Y[2], t.Y[3]);
    t.k = kx | (ky << 8);
    bad |= exp_out(px) | exp_out(py);
    t.ee = (int32_t)px + (int32_t)py;
    if (with_radius) {
        t.rx = __ldg(q.rx + offx);
        t.ry = __ldg(q.ry + offy);
        const int64_t fx = __ldg(q.fx + offx), fy = __ldg(q.fy + offy);
        bad |= exp_out(fx) | exp_out(fy);
        t.s1 = (int32_t)px + (int32_t)fy;
        t.s2 = (int32_t)py + (int32_t)fx;
        t.s3 = (int32_t)fx + (int32_t)fy;
    } else {
        t.rx = t.ry = 0;
        t.s1 = t.s2 = t.s3 = 0;
    }
}

APB_DEV void reg_empty(RTerm& t) {
#pragma unroll
    for (int j = 0; j < 4; j++) t.X[j] = t.Y[j] = 0;
    t.k = 0;  // both kinds APB_ZERO: no contribution, no radius
    t.ee = t.s1 = t.s2 = t.s3 = 0;
    t.rx = t.ry = 0;
}

// special values of a slot: non-finite kinds, infinite radii (Fallback in setup_core)
APB_DEV bool reg_special(const RTerm& t) {
    return (t.k & APB_KIND_MASK) > APB_FINITE || ((t.k >> 8) & APB_KIND_MASK) > APB_FINITE ||
           t.rx == APB_RAD_INF || t.ry == APB_RAD_INF;
}

struct RScan {
    int32_t e_max, e_min, e_rad;  // sentinels INT32_MIN / INT32_MAX / INT32_MIN
    uint32_t nnz;
};

// setup_core over one slot (src/dot.cpp:72-113), special values excluded
APB_DEV void reg_scan(RScan& s, const RTerm& t, bool track_min, bool rad) {
    const uint32_t kx = t.k & APB_KIND_MASK, ky = (t.k >> 8) & APB_KIND_MASK;
    const bool xz = kx == APB_ZERO, yz = ky == APB_ZERO;
    if (!xz && !yz) {
        s.nnz++;
        s.e_max = max(s.e_max, t.ee);
        if (track_min) {  // ApFloat limb counts from the top-aligned slots
            const int cx = (t.X[0] | t.X[1]) ? 2 : 1, cy = (t.Y[0] | t.Y[1]) ? 2 : 1;
            s.e_min = min(s.e_min, t.ee - 64 * (cx + cy));
        }
    }
    if (rad) {
        if (t.ry != 0 && !xz) s.e_rad = max(s.e_rad, t.s1);
        if (t.rx != 0 && !yz) s.e_rad = max(s.e_rad, t.s2);
        if (t.rx != 0 && t.ry != 0) s.e_rad = max(s.e_rad, t.s3);
    }
}

// P = X * Y, 4 x 4 32-bit limbs -> 8: 2 x 2 64-bit limbs with 128-bit partial
// products (IMAD.WIDE.U32 / IMAD.HI chains the compiler schedules freely)
APB_DEV void mul4x4(const uint32_t (&X)[4], const uint32_t (&Y)[4], uint32_t (&P)[8]) {
    const uint64_t a0 = ((uint64_t)X[1] << 32) | X[0], a1 = ((uint64_t)X[3] << 32) | X[2];
    const uint64_t b0 = ((uint64_t)Y[1] << 32) | Y[0], b1 = ((uint64_t)Y[3] << 32) | Y[2];
    const unsigned __int128 p00 = (unsigned __int128)a0 * b0, p01 = (unsigned __int128)a0 * b1;
    const unsigned __int128 p10 = (unsigned __int128)a1 * b0, p11 = (unsigned __int128)a1 * b1;
    const unsigned __int128 mid = (p00 >> 64) + (uint64_t)p01 + (uint64_t)p10;
    const unsigned __int128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + (uint64_t)p11;
    split64((uint64_t)p00, P[0], P[1]);
    split64((uint64_t)mid, P[2], P[3]);
    split64((uint64_t)hi, P[4], P[5]);
    split64((uint64_t)(hi >> 64) + (uint64_t)(p11 >> 64), P[6], P[7]);
}

// (hi:lo) >> t, t in [0, 32)
APB_DEV uint32_t fshr(uint32_t lo, uint32_t hi, uint32_t t) { return __funnelshift_r(lo, hi, t); }

// floor(P / 2^r) into C (2 NSV limbs, the rest 0); returns true iff nonzero bits
// were dropped.  r in [64 (4 - NSV) + ..., 256): q = r / 32 >= q0 = 8 - 2 NSV.
template <int NSV>
APB_DEV bool place(const uint32_t (&P)[8], int r, uint32_t (&C)[6]) {
    constexpr int q0 = 8 - 2 * NSV;
    constexpr int W = 2 * NSV;  // window limbs
    const int q = r >> 5;
    const uint32_t t = (uint32_t)r & 31u;
    uint32_t low = 0;
#pragma unroll
    for (int j = 0; j < q0; j++) low |= P[j];
    if (q <= q0 + 1) {  // the common case: a two-way limb select
        const bool b = q != q0;
        uint32_t Q[W + 1];
#pragma unroll
        for (int k = 0; k <= W; k++) {
            const uint32_t a0 = q0 + k < 8 ? P[q0 + k] : 0u;
            const uint32_t a1 = q0 + 1 + k < 8 ? P[q0 + 1 + k] : 0u;
            Q[k] = b ? a1 : a0;
        }
        low |= b ? P[q0] : 0u;
        low |= t ? (Q[0] << (32 - t)) : 0u;
#pragma unroll
        for (int k = 0; k < W; k++) C[k] = fshr(Q[k], Q[k + 1], t);
    } else {  // far smaller terms: generic limb select
#pragma unroll
        for (int j = q0; j < 8; j++) {
            low |= j < q ? P[j] : 0u;
            low |= (j == q && t) ? (P[j] << (32 - t)) : 0u;
        }
#pragma unroll
        for (int k = 0; k < W; k++) {
            uint32_t lo = 0, hi = 0;
#pragma unroll
            for (int j = q0; j < 8; j++) {
                lo = (j == q + k) ? P[j] : lo;
                hi = (j == q + k + 1) ? P[j] : hi;
            }
            C[k] = fshr(lo, hi, t);
        }
    }
#pragma unroll
    for (int k = W; k < 6; k++) C[k] = 0;
    return low != 0;
}

// a += neg ? -C : C  (mod 2^192), one carry chain: a + (C ^ m) + neg
APB_DEV void acc6(uint32_t (&a)[6], const uint32_t (&C)[6], bool neg) {
    const uint32_t m = neg ? 0xffffffffu : 0u;
    asm("{\n\t.reg .u32 cf;\n\t"
        "add.cc.u32 cf, %6, %6;\n\t"  // carry flag = neg
        "addc.cc.u32 %0, %0, %7;\n\t"
        "addc.cc.u32 %1, %1, %8;\n\t"
        "addc.cc.u32 %2, %2, %9;\n\t"
        "addc.cc.u32 %3, %3, %10;\n\t"
        "addc.cc.u32 %4, %4, %11;\n\t"
        "addc.u32 %5, %5, %12;\n\t}"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5])
        : "r"(m), "r"(C[0] ^ m), "r"(C[1] ^ m), "r"(C[2] ^ m), "r"(C[3] ^ m), "r"(C[4] ^ m), "r"(C[5] ^ m));
}

// a += b (mod 2^192)
APB_DEV void add6(uint32_t (&a)[6], const uint32_t (&b)[6]) {
    asm("add.cc.u32 %0, %0, %6;\n\t"
        "addc.cc.u32 %1, %1, %7;\n\t"
        "addc.cc.u32 %2, %2, %8;\n\t"
        "addc.cc.u32 %3, %3, %9;\n\t"
        "addc.cc.u32 %4, %4, %10;\n\t"
        "addc.u32 %5, %5, %11;"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5])
        : "r"(b[0]), "r"(b[1]), "r"(b[2]), "r"(b[3]), "r"(b[4]), "r"(b[5]));
}

// srad_add (src/dot.cpp:288-295) with the exponent sum s = a.f + b.f precomputed
APB_DEV uint64_t srad_s(uint32_t ab, uint32_t bb, int32_t s, int32_t e_rad) {
    const int32_t d = e_rad - s;
    return d < 30 ? (((uint64_t)ab * bb) >> (30 + d)) + 1 : 1;
}

// one slot of pass 2 (dot_accumulate_term + radius_pass_term), branch-free
// except for the rare far-term limb select inside place()
template <int NSV>
APB_DEV void reg_acc(uint32_t (&a)[6], uint32_t& err, uint64_t& srad, const RTerm& t, int32_t e_s,
                     int32_t e_rad, bool subtract, bool rad) {
    const uint32_t kx = t.k & APB_KIND_MASK, ky = (t.k >> 8) & APB_KIND_MASK;
    const bool xz = kx == APB_ZERO, yz = ky == APB_ZERO;
    const bool nz = !xz && !yz;
    const int32_t sh = e_s - t.ee;
    const bool drop = sh >= 64 * NSV;  // below the window: err only
    uint32_t P[8], C[6];
    mul4x4(t.X, t.Y, P);
    const bool inexact = place<NSV>(P, (drop ? 64 * NSV - 1 : sh) + 256 - 64 * NSV, C);
    const bool use = nz && !drop;
    const uint32_t keep = use ? 0xffffffffu : 0u;
#pragma unroll
    for (int j = 0; j < 6; j++) C[j] &= keep;
    const bool neg = use && (subtract ^ ((t.k & APB_SIGN) != 0) ^ (((t.k >> 8) & APB_SIGN) != 0));
    acc6(a, C, neg);
    err += (nz && (drop || inexact)) ? 1u : 0u;
    if (rad) {
        const uint64_t r1 = srad_s((t.X[3] >> 2) + 1, t.ry, t.s1, e_rad);
        const uint64_t r2 = srad_s((t.Y[3] >> 2) + 1, t.rx, t.s2, e_rad);
        const uint64_t r3 = srad_s(t.rx, t.ry, t.s3, e_rad);
        srad += (t.ry != 0 && !xz) ? r1 : 0;
        srad += (t.rx != 0 && !yz) ? r2 : 0;
        srad += (t.rx != 0 && t.ry != 0) ? r3 : 0;
    }
}

// Mag upper bound of the integer (d2:d1:d0) * 2^base (the window rule of
// mag_upper_of_low_bits, src/apfloat.cpp:26-63: top 30 bits, +1 if any bit
// below them is set; exponent base + bit length)
APB_DEV Mag mag_upper192(uint64_t d0, uint64_t d1, uint64_t d2, int64_t base) {
    if (!(d0 | d1 | d2)) return mag_zero();
    const int lz = d2 ? __clzll((long long)d2) : d1 ? 64 + __clzll((long long)d1) : 128 + __clzll((long long)d0);
    // top 64 bits of the value and a sticky bit for everything below
    uint64_t top, rest;
    if (lz < 64) {
        top = lz ? (d2 << lz) | (d1 >> (64 - lz)) : d2;
        rest = (lz ? d1 << lz : d1) | d0;
    } else if (lz < 128) {
        const int l = lz - 64;
        top = l ? (d1 << l) | (d0 >> (64 - l)) : d1;
        rest = l ? d0 << l : d0;
    } else {
        top = d0 << (lz - 128);
        rest = 0;
    }
    uint64_t b = top >> 34;
    if (rest || (top & ((1ull << 34) - 1))) b++;
    return mag_parts(b, base + (192 - lz));
}

// dot_finalize (src/dot.cpp:306-321) for n_s <= 3 in registers: sign fix
// (neg_in_place), apfloat_normalize as a 192-bit left shift, apfloat_round as a
// mask of the bits below the top p, then rad = round_err + err ulps + srad
// (src/mag.cpp:108-130 order); same results as finalize_store<3>.
APB_DEV void finalize_fast(const Plan& pl, uint64_t s0, uint64_t s1, uint64_t s2, uint64_t err, uint64_t srad,
                           int64_t prec, bool with_radius, const BallsOut& out, int64_t b, int* status) {
    int64_t p = prec > pl.p_eff ? pl.p_eff : prec;
    if (p < 2) p = 2;
    const bool three = pl.n_s == 3;
    if (!three) s2 = 0;
    const bool sign = (three ? s2 : s1) >> 63;
    if (sign) {  // two's complement negation mod 2^(64 n_s)
        s0 = ~s0;
        s1 = ~s1;
        s2 = three ? ~s2 : 0;
        asm("add.cc.u64 %0, %0, 1;\n\taddc.cc.u64 %1, %1, 0;\n\taddc.u64 %2, %2, 0;"
            : "+l"(s0), "+l"(s1), "+l"(s2));
        if (!three) s2 = 0;
    }
    uint64_t* dst = out.mant + b * (int64_t)out.L;
    Mag r = mag_zero();
    if (!(s0 | s1 | s2)) {
        for (int i = 0; i < out.L; i++) dst[i] = 0;
        out.exp[b] = 0;
        out.kind[b] = APB_ZERO;
    } else {
        const int lz = s2 ? __clzll((long long)s2) : s1 ? 64 + __clzll((long long)s1) : 128 + __clzll((long long)s0);
        const int64_t e = pl.e_s - 64 * (int64_t)pl.n_s + (192 - lz);
        // W = V << lz, top-aligned in three limbs
        uint64_t w0 = s0, w1 = s1, w2 = s2;
        if (lz >= 128) {
            w2 = s0;
            w1 = 0;
            w0 = 0;
        } else if (lz >= 64) {
            w2 = s1;
            w1 = s0;
            w0 = 0;
        }
        const int l = lz & 63;
        if (l) {
            w2 = (w2 << l) | (w1 >> (64 - l));
            w1 = (w1 << l) | (w0 >> (64 - l));
            w0 <<= l;
        }
        // truncate to p bits: D = W mod 2^(192 - p) is the rounding error
        if (p < 192) {
            const int c = 192 - (int)p;  // bits cut, in (0, 190]
            uint64_t m0 = c >= 64 ? ~0ull : ((1ull << c) - 1);
            uint64_t m1 = c >= 128 ? ~0ull : (c > 64 ? ((1ull << (c - 64)) - 1) : 0ull);
            uint64_t m2 = c > 128 ? ((1ull << (c - 128)) - 1) : 0ull;
            r = mag_upper192(w0 & m0, w1 & m1, w2 & m2, e - 192);
            w0 &= ~m0;
            w1 &= ~m1;
            w2 &= ~m2;
        }
        const int L = out.L;
        for (int i = 0; i < L - 3; i++) dst[i] = 0;
        if (L >= 3) dst[L - 3] = w0;
        else if (w0) *status = APB_ERR_UNSUPPORTED;
        if (L >= 2) dst[L - 2] = w1;
        else if (w1) *status = APB_ERR_UNSUPPORTED;
        dst[L - 1] = w2;
        out.exp[b] = e;
        out.kind[b] = (uint8_t)(APB_FINITE | (sign ? APB_SIGN : 0));
    }
    if (with_radius) {
        if (err) r = mag_add(r, mag_from_u64(err, pl.e_s - 64 * (int64_t)pl.n_s));
        if (srad) r = mag_add(r, mag_from_u64(srad, pl.e_rad - 30));
    } else {
        r = mag_zero();
    }
    mag_store(r, &out.rad_man[b], &out.rad_exp[b]);
}

// group (TPD lanes) reductions of 32-bit values (redux.sync for whole warps)
template <int TPD>
APB_DEV int32_t grp_max32(int32_t v) {
    if (TPD == 32) return __reduce_max_sync(0xffffffffu, v);
#pragma unroll
    for (int o = TPD / 2; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int TPD>
APB_DEV int32_t grp_min32(int32_t v) {
    if (TPD == 32) return __reduce_min_sync(0xffffffffu, v);
#pragma unroll
    for (int o = TPD / 2; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <int TPD>
APB_DEV uint32_t grp_add32(uint32_t v) {
    if (TPD == 32) return __reduce_add_sync(0xffffffffu, v);
#pragma unroll
    for (int o = TPD / 2; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <int TPD>
APB_DEV uint32_t grp_or32(uint32_t v) {
    if (TPD == 32) return __reduce_or_sync(0xffffffffu, v);
#pragma unroll
    for (int o = TPD / 2; o; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// prefetch the 128-byte lines holding [p, p + bytes) into L2 (lanes over the lines)
APB_DEV void pf_range(const void* p, int64_t bytes, int lane) {
    const char* c = (const char*)p;
    for (int64_t j = (int64_t)lane * 128; j < bytes + 127; j += 32 * 128) {
        const char* a = c + (j < bytes ? j : bytes - 1);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
}

#ifndef APB_REG_MINB
#define APB_REG_MINB 3
#endif

// TPD lanes per dot, RS register slots per lane (n <= TPD * RS); a warp runs
// 32 / TPD dots side by side and walks its dot groups round-robin over the
// grid (persistent); reduced states are parked and finalized 32 at a time.
// UNIT: xstep == ystep == 1 (slot offsets are compile-time constants); PF: flat
// contiguous dots (bdiv = 1, xs1 = ys1 = n), whose next group is prefetched into L2.
template <int TPD, int RS, bool UNIT, bool PF>
__global__ void __launch_bounds__(128, APB_REG_MINB) dot_reg_kernel(DotArgs A, int64_t ngroups) {
    constexpr int DPR = 32 / TPD;
    constexpr int PK = 11;  // s[3], err, srad, e_max, e_min, e_rad, nnz, flags, dot index
    __shared__ uint64_t park[4][32][PK];
    const int lane = threadIdx.x & 31, sub = lane % TPD, grp = lane / TPD, wl = threadIdx.x >> 5;
    const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const bool with_radius = A.mode == APB_DOT_BALL;
    const bool track_min = A.prec > 128;
    const bool subtract = A.subtract != 0;
    int parked = 0;
    for (int64_t g = (int64_t)blockIdx.x * (blockDim.x >> 5) + wl; g < ngroups; g += nwarps) {
        const int64_t b = g * DPR + grp;
        const bool live = b < A.batch;
        int64_t ex0 = 0, xst = 0, ey0 = 0, yst = 0, nb = 0;
        if (live) dot_extent(A, b, ex0, xst, ey0, yst, nb);
        ex0 += sub * xst;
        ey0 += sub * yst;
        RPtrs q;
        q.kx = A.x.kind + ex0;
        q.ky = A.y.kind + ey0;
        q.ex = A.x.exp + ex0;
        q.ey = A.y.exp + ey0;
        q.fx = A.x.rad_exp + ex0;
        q.fy = A.y.rad_exp + ey0;
        q.rx = A.x.rad_man + ex0;
        q.ry = A.y.rad_man + ey0;
        q.mx = A.x.mant + ex0 * (A.mant16 ? 2 : A.x.L);
        q.my = A.y.mant + ey0 * (A.mant16 ? 2 : A.y.L);
        // ---- L2 prefetch of the warp's next dot group (contiguous unit-stride
        // dots): its loads then wait on L2, not DRAM
        if (PF && g + nwarps < ngroups) {
            const int64_t b2 = (g + nwarps) * DPR;
            const int64_t nd2 = min((int64_t)DPR, A.batch - b2);
            const int64_t e2x = A.idx.x_off + b2 * A.idx.xs1, e2y = A.idx.y_off + b2 * A.idx.ys1;
            const int64_t cnt = (nd2 - 1) * A.idx.xs1 + A.n;  // elements spanned (xs1 == ys1 == n here)
            pf_range(A.x.mant + e2x * A.x.L, cnt * 8 * A.x.L, lane);
            pf_range(A.y.mant + e2y * A.y.L, cnt * 8 * A.y.L, lane);
            pf_range(A.x.exp + e2x, cnt * 8, lane);
            pf_range(A.y.exp + e2y, cnt * 8, lane);
            pf_range(A.x.kind + e2x, cnt, lane);
            pf_range(A.y.kind + e2y, cnt, lane);
            if (with_radius) {
                pf_range(A.x.rad_exp + e2x, cnt * 8, lane);
                pf_range(A.y.rad_exp + e2y, cnt * 8, lane);
                pf_range(A.x.rad_man + e2x, cnt * 4, lane);
                pf_range(A.y.rad_man + e2y, cnt * 4, lane);
            }
        }
        // ---- one load of the dot's terms into registers (RS = ceil(n / TPD):
        // slots 0..RS-2 are full, the last one reads a clamped element and masks it)
        RTerm t[RS];
        uint32_t bad = 0;
        if (nb > 0) {
#pragma unroll
            for (int k = 0; k < RS; k++) {
                if (k < RS - 1) {
                    const int64_t ox = UNIT ? (int64_t)k * TPD : (int64_t)k * TPD * xst;
                    const int64_t oy = UNIT ? (int64_t)k * TPD : (int64_t)k * TPD * yst;
                    reg_load(t[k], A, q, ox, oy, with_radius, bad);
                } else {
                    const int64_t i = sub + (int64_t)k * TPD;
                    const int64_t ic = (i < nb ? i : nb - 1) - sub;
                    reg_load(t[k], A, q, UNIT ? ic : ic * xst, UNIT ? ic : ic * yst, with_radius, bad);
                    if (i >= nb) {
                        t[k].k = 0;
                        t[k].rx = t[k].ry = 0;
                    }
                }
            }
        } else {
#pragma unroll
            for (int k = 0; k < RS; k++) reg_empty(t[k]);
        }
        // ---- pass 1: setup scan; exceptional dots (special values, exponents
        // beyond 2^29) go to the generic kernel
        uint32_t any_rad = 0;
#pragma unroll
        for (int k = 0; k < RS; k++) {
            bad |= reg_special(t[k]) ? 1u : 0u;
            any_rad |= t[k].rx | t[k].ry;
        }
        const bool exc = grp_or32<TPD>(bad) != 0;
        const bool rad = with_radius && grp_or32<TPD>(any_rad) != 0;
        RScan sc{INT32_MIN, INT32_MAX, INT32_MIN, 0};
#pragma unroll
        for (int k = 0; k < RS; k++) reg_scan(sc, t[k], track_min, rad);
        sc.nnz = grp_add32<TPD>(sc.nnz);
        sc.e_max = grp_max32<TPD>(sc.e_max);
        if (track_min) sc.e_min = grp_min32<TPD>(sc.e_min);
        if (rad) sc.e_rad = grp_max32<TPD>(sc.e_rad);
        const int64_t e_max64 = sc.e_max == INT32_MIN ? INT64_MIN : (int64_t)sc.e_max;
        const int64_t e_min64 = sc.e_min == INT32_MAX ? INT64_MAX : (int64_t)sc.e_min;
        const int64_t e_rad64 = sc.e_rad == INT32_MIN ? INT64_MIN : (int64_t)sc.e_rad;
        const Plan pl = finish_plan(e_max64, e_min64, e_rad64, sc.nnz, exc, nb, A.prec, A.disable_reduction);
        // ---- pass 2: accumulate
        uint32_t a[6] = {0, 0, 0, 0, 0, 0};
        uint32_t err = 0;
        uint64_t srad = 0;
        if (live && pl.status == 0) {
            const int32_t e_s = (int32_t)pl.e_s, e_rad = sc.e_rad;
            if (pl.n_s == 3) {
#pragma unroll
                for (int k = 0; k < RS; k++) reg_acc<3>(a, err, srad, t[k], e_s, e_rad, subtract, rad);
            } else {
#pragma unroll
                for (int k = 0; k < RS; k++) reg_acc<2>(a, err, srad, t[k], e_s, e_rad, subtract, rad);
            }
        }
        // ---- group reduction (carry chain mod 2^192)
#pragma unroll
        for (int o = TPD / 2; o; o >>= 1) {
            uint32_t v[6];
#pragma unroll
            for (int j = 0; j < 6; j++) v[j] = __shfl_xor_sync(0xffffffffu, a[j], o);
            add6(a, v);
        }
        err = grp_add32<TPD>(err);
        if (rad) {
#pragma unroll
            for (int o = TPD / 2; o; o >>= 1) srad += __shfl_xor_sync(0xffffffffu, srad, o);
        }
        // ---- park (group leader); empty records for groups past the batch
        if (sub == 0) {
            uint64_t* pk = park[wl][parked + grp];
            pk[0] = (uint64_t)a[0] | ((uint64_t)a[1] << 32);
            pk[1] = (uint64_t)a[2] | ((uint64_t)a[3] << 32);
            pk[2] = (uint64_t)a[4] | ((uint64_t)a[5] << 32);
            pk[3] = err;
            pk[4] = srad;
            pk[5] = (uint64_t)e_max64;
            pk[6] = (uint64_t)e_min64;
            pk[7] = (uint64_t)e_rad64;
            pk[8] = sc.nnz;
            pk[9] = exc ? 1 : 0;
            pk[10] = live ? (uint64_t)b : ~0ull;
        }
        parked += DPR;
        const bool last = g + nwarps >= ngroups;
        if (parked + DPR > 32 || last) {
            __syncwarp();
            const int np = parked;
            if (lane < np) {
                const uint64_t* pk = park[wl][lane];
                const int64_t bb = (int64_t)pk[10];
                if ((uint64_t)bb < (uint64_t)A.batch) {
                    if (pk[9]) {  // recomputed by dot_generic_kernel (fallback_only pass)
                        A.fb_flag[bb] = 1;
                    } else {
                        int64_t e0, s0, f0, u0, n0;
                        dot_extent(A, bb, e0, s0, f0, u0, n0);
                        const Plan fp = finish_plan((int64_t)pk[5], (int64_t)pk[6], (int64_t)pk[7], pk[8], false,
                                                    n0, A.prec, A.disable_reduction);
                        if (fp.status != 0) {  // ZeroResult
                            if (A.state) write_state(A.state + bb, fp, 0, 0);
                            GFloat<1> z;
                            z.kind = APB_ZERO;
                            z.neg = 0;
                            z.e = 0;
                            z.n = 0;
                            gf_store(A.out, bb, z, mag_zero(), A.status);
                        } else {
                            uint64_t s3[3] = {pk[0], pk[1], pk[2]};
                            if (A.state) write_state(A.state + bb, fp, pk[3], pk[4]);
                            if (A.acc)
                                for (int j = 0; j < fp.n_s && j < A.acc_stride; j++)
                                    A.acc[bb * A.acc_stride + j] = s3[j];
                            finalize_fast(fp, s3[0], s3[1], s3[2], pk[3], pk[4], A.prec, with_radius, A.out, bb, A.status);
                        }
                    }
                }
            }
            __syncwarp();
            parked = 0;
        }
    }
}
