// apb_common.cuh - device-side number primitives shared by the dot and matmul
// kernels: Mag upper-bound arithmetic (reference include/apball/mag.hpp,
// src/mag.cpp), limb helpers, and a bounded-size generic float used by the
// rare paths (finalize, special-value fallback).  Paths are relative to
// /root/reference/proj.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "apb.h"

#define APB_DEV __device__ __forceinline__

namespace apb {

// ------------------------------------------------------------------ limbs

APB_DEV unsigned bitw64(uint64_t v) { return v ? 64u - (unsigned)__clzll((long long)v) : 0u; }
APB_DEV unsigned ctz64(uint64_t v) { return (unsigned)__ffsll((long long)v) - 1u; }

// programmatic dependent launch (launch_pdl in apb_internal.h): wait for the
// stream predecessor's completion and memory flush / let dependents launch early.
// Both are no-ops for kernels launched without the attribute.
APB_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
APB_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// (lo >> rb) | (hi << (64-rb)), rb in [0,64)
APB_DEV uint64_t funnel_r(uint64_t lo, uint64_t hi, unsigned rb) {
    return rb ? (lo >> rb) | (hi << (64 - rb)) : lo;
}

// s += c / s -= c modulo 2^(64 NS), one PTX carry chain (add.cc / addc) for
// the small window widths of the dot kernels, a compare-and-carry loop otherwise
template <int NS>
APB_DEV void addn_mod(uint64_t (&s)[NS], const uint64_t (&c)[NS]) {
    if constexpr (NS == 2) {
        asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(s[0]), "+l"(s[1]) : "l"(c[0]), "l"(c[1]));
    } else if constexpr (NS == 3) {
        asm("add.cc.u64 %0, %0, %3;\n\taddc.cc.u64 %1, %1, %4;\n\taddc.u64 %2, %2, %5;"
            : "+l"(s[0]), "+l"(s[1]), "+l"(s[2]) : "l"(c[0]), "l"(c[1]), "l"(c[2]));
    } else if constexpr (NS == 5) {
        asm("add.cc.u64 %0, %0, %5;\n\taddc.cc.u64 %1, %1, %6;\n\taddc.cc.u64 %2, %2, %7;\n\t"
            "addc.cc.u64 %3, %3, %8;\n\taddc.u64 %4, %4, %9;"
            : "+l"(s[0]), "+l"(s[1]), "+l"(s[2]), "+l"(s[3]), "+l"(s[4])
            : "l"(c[0]), "l"(c[1]), "l"(c[2]), "l"(c[3]), "l"(c[4]));
    } else {
        uint64_t cy = 0;
#pragma unroll
        for (int j = 0; j < NS; j++) {
            const uint64_t s1 = s[j] + c[j];
            const uint64_t c1 = s1 < c[j];
            const uint64_t s2 = s1 + cy;
            cy = c1 | (s2 < cy);
            s[j] = s2;
        }
    }
}
template <int NS>
APB_DEV void subn_mod(uint64_t (&s)[NS], const uint64_t (&c)[NS]) {
    if constexpr (NS == 2) {
        asm("sub.cc.u64 %0, %0, %2;\n\tsubc.u64 %1, %1, %3;" : "+l"(s[0]), "+l"(s[1]) : "l"(c[0]), "l"(c[1]));
    } else if constexpr (NS == 3) {
        asm("sub.cc.u64 %0, %0, %3;\n\tsubc.cc.u64 %1, %1, %4;\n\tsubc.u64 %2, %2, %5;"
            : "+l"(s[0]), "+l"(s[1]), "+l"(s[2]) : "l"(c[0]), "l"(c[1]), "l"(c[2]));
    } else if constexpr (NS == 5) {
        asm("sub.cc.u64 %0, %0, %5;\n\tsubc.cc.u64 %1, %1, %6;\n\tsubc.cc.u64 %2, %2, %7;\n\t"
            "subc.cc.u64 %3, %3, %8;\n\tsubc.u64 %4, %4, %9;"
            : "+l"(s[0]), "+l"(s[1]), "+l"(s[2]), "+l"(s[3]), "+l"(s[4])
            : "l"(c[0]), "l"(c[1]), "l"(c[2]), "l"(c[3]), "l"(c[4]));
    } else {
        uint64_t bw = 0;
#pragma unroll
        for (int j = 0; j < NS; j++) {
            const uint64_t x = s[j], y = c[j];
            s[j] = x - y - bw;
            bw = (x < y) || (x == y && bw);
        }
    }
}

// 64x64 -> 128
APB_DEV void mul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
    lo = a * b;
    hi = __umul64hi(a, b);
}

// ------------------------------------------------------------------- Mag
// (b / 2^30) * 2^f, 2^29 <= b < 2^30 (include/apball/mag.hpp:15-59)
struct Mag {
    int kind;  // 0 zero, 1 finite, 2 inf
    uint64_t b;
    int64_t f;
};

constexpr uint64_t kMagOne = 1ull << 30;
constexpr int64_t kMExpMax = INT64_MAX - 4;
constexpr int64_t kMExpMin = INT64_MIN + 4;

APB_DEV Mag mag_zero() { return Mag{0, 0, 0}; }
APB_DEV Mag mag_inf() { return Mag{2, 0, 0}; }

// Mag::from_parts (src/mag.cpp:18-31)
APB_DEV Mag mag_parts(uint64_t b, int64_t f) {
    if (b == kMagOne) {
        b = kMagOne >> 1;
        if (f >= kMExpMax) return mag_inf();
        f++;
    }
    return Mag{1, b, f};
}

// Mag::from_u64_upper (src/mag.cpp:33-50)
APB_DEV Mag mag_from_u64(uint64_t v, int64_t exp2) {
    if (v == 0) return mag_zero();
    unsigned len = bitw64(v);
    uint64_t b;
    bool inexact = false;
    if (len <= 30) {
        b = v << (30 - len);
    } else {
        unsigned sh = len - 30;
        b = v >> sh;
        inexact = (v & ((1ull << sh) - 1)) != 0;
    }
    if (inexact) b++;
    // exp2 + len in 128-bit-safe form
    if (exp2 > kMExpMax - (int64_t)len) return mag_inf();
    int64_t f = exp2 + (int64_t)len;
    if (f < kMExpMin) return mag_parts(kMagOne >> 1, kMExpMin);
    return mag_parts(b, f);
}

// Mag::from_double_upper (src/mag.cpp:79-87)
APB_DEV Mag mag_from_double(double v, int64_t exp2) {
    if (v == 0.0) return mag_zero();
    if (isinf(v) || isnan(v)) return mag_inf();
    int e;
    double fr = frexp(v, &e);
    uint64_t m53 = (uint64_t)ldexp(fr, 53);
    return mag_from_u64(m53, exp2 + e - 53);
}

APB_DEV int mag_cmp(const Mag& a, const Mag& b) {
    int ra = a.kind == 0 ? 0 : (a.kind == 2 ? 2 : 1);
    int rb = b.kind == 0 ? 0 : (b.kind == 2 ? 2 : 1);
    if (ra != rb || ra != 1) return ra < rb ? -1 : (ra > rb ? 1 : 0);
    if (a.f != b.f) return a.f < b.f ? -1 : 1;
    if (a.b != b.b) return a.b < b.b ? -1 : 1;
    return 0;
}

// mag_add_up (src/mag.cpp:108-130)
APB_DEV Mag mag_add(const Mag& a, const Mag& b) {
    if (a.kind == 2 || b.kind == 2) return mag_inf();
    if (a.kind == 0) return b;
    if (b.kind == 0) return a;
    Mag hi = a, lo = b;
    if (mag_cmp(hi, lo) < 0) {
        hi = b;
        lo = a;
    }
    uint64_t bh = hi.b;
    int64_t f = hi.f;
    uint64_t d = (uint64_t)(f - lo.f);
    if (d >= 30) {
        bh += 1;
    } else {
        uint64_t bl = lo.b;
        bh += bl >> d;
        if (d && (bl & ((1ull << d) - 1))) bh++;
    }
    while (bh > kMagOne) {
        bh = (bh + 1) >> 1;
        if (f >= kMExpMax) return mag_inf();
        f++;
    }
    return mag_parts(bh, f);
}

// mag_mul_up (src/mag.cpp:132-145)
APB_DEV Mag mag_mul(const Mag& a, const Mag& b) {
    if (a.kind == 0 || b.kind == 0) return mag_zero();
    if (a.kind == 2 || b.kind == 2) return mag_inf();
    uint64_t p = a.b * b.b;
    uint64_t q = (p + (kMagOne - 1)) >> 30;
    // f = a.f + b.f with saturation
    __int128 f = (__int128)a.f + b.f;
    if (q < (kMagOne >> 1)) {
        q <<= 1;
        f--;
    }
    if (f > kMExpMax) return mag_inf();
    if (f < kMExpMin) return mag_parts(kMagOne >> 1, kMExpMin);
    return mag_parts(q, (int64_t)f);
}

APB_DEV Mag mag_load(uint32_t b, int64_t f) {
    if (b == 0) return mag_zero();
    if (b == APB_RAD_INF) return mag_inf();
    return mag_parts(b, f);
}

APB_DEV void mag_store(const Mag& r, uint32_t* man, int64_t* ex) {
    if (r.kind == 0) {
        *man = 0;
        *ex = 0;
    } else if (r.kind == 2) {
        *man = APB_RAD_INF;
        *ex = 0;
    } else {
        *man = (uint32_t)r.b;
        *ex = r.f;
    }
}

// ----------------------------------------------------------- ball arrays

struct BallsView {
    const uint64_t* mant;
    const int64_t* exp;
    const uint8_t* kind;
    const uint32_t* rad_man;
    const int64_t* rad_exp;
    int32_t L;
};

struct BallsOut {
    uint64_t* mant;
    int64_t* exp;
    uint8_t* kind;
    uint32_t* rad_man;
    int64_t* rad_exp;
    int32_t L;
};

inline BallsView view_of(const apb_balls* a) {
    return BallsView{a->mant, a->exp, a->kind, a->rad_man, a->rad_exp, a->L};
}
inline BallsOut out_of(apb_balls* a) {
    return BallsOut{a->mant, a->exp, a->kind, a->rad_man, a->rad_exp, a->L};
}

// ------------------------------------------------ bounded generic float
// A finite/special float with up to CAP limbs, used by finalize and the
// special-value fallback.  Restates apfloat_normalize / apfloat_round /
// apfloat_add_round / apfloat_mul_exact (src/apfloat.cpp:116-270).

template <int CAP>
struct GFloat {
    int kind;  // APB_ZERO .. APB_NAN
    int neg;
    int64_t e;
    int n;
    uint64_t d[CAP];
};

constexpr int64_t kExpHi = INT64_MAX - 8;
constexpr int64_t kExpLo = INT64_MIN + 8;

// e + a (a small) with the reference's overflow_error semantics
APB_DEV int64_t checked_add(int64_t e, int64_t a, int* status) {
    __int128 r = (__int128)e + a;
    if (r > kExpHi || r < kExpLo) {
        *status = APB_ERR_OVERFLOW;
        return 0;
    }
    return (int64_t)r;
}

// apfloat_normalize (src/apfloat.cpp:116-136): value = (-1)^neg 2^e raw/2^(64 nraw)
template <int CAP>
__device__ void gf_normalize(GFloat<CAP>& out, int neg, int64_t e, const uint64_t* raw, int nraw,
                             int* status) {
    int h = nraw;
    while (h > 0 && raw[h - 1] == 0) h--;
    if (h == 0) {
        out.kind = APB_ZERO;
        out.neg = 0;
        out.e = 0;
        out.n = 0;
        return;
    }
    unsigned tb = bitw64(raw[h - 1]);
    int64_t adj = -64 * (int64_t)nraw + 64 * (int64_t)(h - 1) + (int64_t)tb;
    int64_t e_new = checked_add(e, adj, status);
    unsigned sh = (64 - tb) % 64;
    for (int i = h - 1; i >= 0; i--)
        out.d[i] = sh ? ((raw[i] << sh) | (i > 0 ? raw[i - 1] >> (64 - sh) : 0)) : raw[i];
    int z = 0;
    while (out.d[z] == 0) z++;
    int cnt = h - z;
    if (z)
        for (int i = 0; i < cnt; i++) out.d[i] = out.d[i + z];
    out.kind = APB_FINITE;
    out.neg = neg;
    out.e = e_new;
    out.n = cnt;
}

// mag_upper_of_low_bits (src/apfloat.cpp:26-63)
APB_DEV Mag mag_low_bits(const uint64_t* limbs, int cut_limbs, unsigned cut_bits, int64_t base,
                         int* status) {
    int t = -1;
    uint64_t tv = 0;
    if (cut_bits) {
        uint64_t part = limbs[cut_limbs] & ((1ull << cut_bits) - 1);
        if (part) {
            t = cut_limbs;
            tv = part;
        }
    }
    if (t < 0) {
        for (int i = cut_limbs - 1; i >= 0; i--)
            if (limbs[i]) {
                t = i;
                tv = limbs[i];
                break;
            }
    }
    if (t < 0) return mag_zero();
    unsigned tb = bitw64(tv);
    uint64_t window = tb < 64 ? tv << (64 - tb) : tv;
    bool low = false;
    if (t > 0) {
        if (tb < 64) {
            window |= limbs[t - 1] >> tb;
            if (limbs[t - 1] & ((1ull << tb) - 1)) low = true;
        } else if (limbs[t - 1]) {
            low = true;
        }
        for (int i = 0; i + 1 < t && !low; i++)
            if (limbs[i]) low = true;
    }
    uint64_t b = window >> 34;
    if (low || (window & ((1ull << 34) - 1))) b++;
    return mag_parts(b, checked_add(base, 64 * (int64_t)t + (int64_t)tb, status));
}

// apfloat_round (src/apfloat.cpp:138-162), in place; returns the error Mag
template <int CAP>
__device__ Mag gf_round(GFloat<CAP>& x, int64_t p, int* status) {
    if (x.kind != APB_FINITE) return mag_zero();
    const int n = x.n;
    if (p >= 64 * (int64_t)n) return mag_zero();
    const int64_t cut = 64 * (int64_t)n - p;
    const int cut_limbs = (int)(cut / 64);
    const unsigned cut_bits = (unsigned)(cut % 64);
    Mag err = mag_low_bits(x.d, cut_limbs, cut_bits, x.e - 64 * (int64_t)n, status);
    if (err.kind == 0) return err;
    int keep = n - cut_limbs;
    for (int i = 0; i < keep; i++) x.d[i] = x.d[i + cut_limbs];
    if (cut_bits) x.d[0] &= ~((1ull << cut_bits) - 1);
    int z = 0;
    while (x.d[z] == 0) z++;
    if (z) {
        for (int i = 0; i + z < keep; i++) x.d[i] = x.d[i + z];
    }
    x.n = keep - z;
    return err;
}

// store a generic float + Mag into slot e of an output ball array
template <int CAP>
__device__ void gf_store(const BallsOut& o, int64_t e, const GFloat<CAP>& m, const Mag& r,
                         int* status) {
    uint64_t* dst = o.mant + e * (int64_t)o.L;
    for (int i = 0; i < o.L; i++) dst[i] = 0;
    o.exp[e] = 0;
    o.kind[e] = (uint8_t)m.kind;
    if (m.kind == APB_FINITE) {
        if (m.n > o.L) {
            *status = APB_ERR_UNSUPPORTED;
        } else {
            for (int i = 0; i < m.n; i++) dst[o.L - m.n + i] = m.d[i];
        }
        o.exp[e] = m.e;
        if (m.neg) o.kind[e] |= APB_SIGN;
    }
    mag_store(r, &o.rad_man[e], &o.rad_exp[e]);
}

// load slot e of a ball array as a generic float (limb count = minimal)
template <int CAP>
__device__ void gf_load(GFloat<CAP>& x, const BallsView& a, int64_t e) {
    uint8_t k = a.kind[e];
    x.kind = k & APB_KIND_MASK;
    x.neg = x.kind == APB_NINF;
    x.e = 0;
    x.n = 0;
    if (x.kind != APB_FINITE) return;
    const uint64_t* m = a.mant + e * (int64_t)a.L;
    int z = 0;
    while (z < a.L && m[z] == 0) z++;
    x.n = a.L - z;
    for (int i = 0; i < x.n; i++) x.d[i] = m[z + i];
    x.e = a.exp[e];
    x.neg = (k & APB_SIGN) != 0;
}

// ----------------------------------------- generic arithmetic (bounded)

constexpr int GCAP = 140;  // limbs: p <= 4096 inputs (64 limbs) and n_s <= 136

typedef GFloat<GCAP> GF;

// apfloat_mul_exact (src/apfloat.cpp:164-176)
__device__ inline void gf_mul_exact(GF& out, const GF& a, const GF& b, int* status) {
    if (a.kind == APB_NAN || b.kind == APB_NAN) {
        out.kind = APB_NAN;
        out.neg = 0;
        out.n = 0;
        out.e = 0;
        return;
    }
    const bool ai = a.kind == APB_PINF || a.kind == APB_NINF;
    const bool bi = b.kind == APB_PINF || b.kind == APB_NINF;
    if (ai || bi) {
        out.n = 0;
        out.e = 0;
        if (a.kind == APB_ZERO || b.kind == APB_ZERO) {
            out.kind = APB_NAN;
            out.neg = 0;
            return;
        }
        const int sa = a.kind == APB_NINF || (a.kind == APB_FINITE && a.neg);
        const int sb = b.kind == APB_NINF || (b.kind == APB_FINITE && b.neg);
        out.kind = sa != sb ? APB_NINF : APB_PINF;
        out.neg = sa != sb;
        return;
    }
    if (a.kind == APB_ZERO || b.kind == APB_ZERO) {
        out.kind = APB_ZERO;
        out.neg = 0;
        out.n = 0;
        out.e = 0;
        return;
    }
    uint64_t prod[2 * GCAP];
    for (int k = 0; k < a.n + b.n; k++) prod[k] = 0;
    for (int j = 0; j < b.n; j++) {
        uint64_t cy = 0;
        for (int i = 0; i < a.n; i++) {
            uint64_t lo, hi;
            mul64(a.d[i], b.d[j], lo, hi);
            uint64_t s1 = prod[i + j] + lo;
            uint64_t c1 = s1 < lo;
            uint64_t s2 = s1 + cy;
            uint64_t c2 = s2 < cy;
            prod[i + j] = s2;
            cy = hi + c1 + c2;
        }
        prod[a.n + j] = cy;
    }
    int64_t e = checked_add(a.e, b.e, status);
    gf_normalize(out, a.neg != b.neg, e, prod, a.n + b.n, status);
}

// place_truncated (src/apfloat.cpp:197-224)
__device__ inline int place_trunc(uint64_t* out, const GF& x, int64_t win_bot) {
    const int n = x.n;
    // off = e - 64n - win_bot, computed without overflow for the values that occur
    const int64_t off = (x.e - 64 * (int64_t)n) - win_bot;
    if (off >= 0) {
        int ol = (int)(off / 64);
        unsigned sh = (unsigned)(off % 64);
        for (int i = 0; i < n; i++) {
            out[ol + i] |= x.d[i] << sh;
            if (sh) out[ol + i + 1] |= x.d[i] >> (64 - sh);
        }
        return 0;
    }
    const int64_t drop = -off;
    const int64_t dl = drop / 64;
    const unsigned db = (unsigned)(drop % 64);
    if (dl >= n) return 1;
    int inexact = db && (x.d[dl] & ((1ull << db) - 1));
    for (int i = 0; i < dl && !inexact; i++)
        if (x.d[i]) inexact = 1;
    for (int i = (int)dl; i < n; i++) {
        uint64_t v = db ? x.d[i] >> db : x.d[i];
        if (db && i + 1 < n) v |= x.d[i + 1] << (64 - db);
        out[i - dl] = v;
    }
    return inexact;
}

// apfloat_add_round (src/apfloat.cpp:228-270); res may alias a
__device__ inline Mag gf_add_round(GF& res, const GF& a, const GF& b, int64_t p, int* status) {
    if (p < 2) p = 2;
    if (a.kind == APB_NAN || b.kind == APB_NAN) {
        res.kind = APB_NAN;
        res.neg = 0;
        res.n = 0;
        res.e = 0;
        return mag_zero();
    }
    const bool ai = a.kind == APB_PINF || a.kind == APB_NINF;
    const bool bi = b.kind == APB_PINF || b.kind == APB_NINF;
    if (ai || bi) {
        if (ai && bi) {
            if (a.kind == b.kind) {
                if (&res != &a) res = a;
            } else {
                res.kind = APB_NAN;
                res.neg = 0;
                res.n = 0;
                res.e = 0;
            }
        } else {
            if (ai) {
                if (&res != &a) res = a;
            } else {
                res = b;
            }
        }
        return mag_zero();
    }
    if (a.kind == APB_ZERO) {
        res = b;
        return gf_round(res, p, status);
    }
    if (b.kind == APB_ZERO) {
        if (&res != &a) res = a;
        return gf_round(res, p, status);
    }
    const int64_t e_top = (a.e > b.e ? a.e : b.e) + 1;
    const int64_t bot_a = a.e - 64 * (int64_t)a.n;
    const int64_t bot_b = b.e - 64 * (int64_t)b.n;
    const int64_t span = e_top - (bot_a < bot_b ? bot_a : bot_b);
    int64_t k = (span + 63) / 64;
    const int64_t budget = p / 64 + 3;
    if (k > budget) k = budget;
    const int64_t win_bot = checked_add(e_top, -64 * k, status);
    uint64_t Aw[GCAP + 2], Bw[GCAP + 2], S[GCAP + 2];
    for (int i = 0; i <= k; i++) Aw[i] = Bw[i] = 0;
    unsigned units = 0;
    units += place_trunc(Aw, a, win_bot);
    units += place_trunc(Bw, b, win_bot);
    int sign;
    int cmp = 0;
    for (int i = (int)k; i >= 0; i--)
        if (Aw[i] != Bw[i]) {
            cmp = Aw[i] > Bw[i] ? 1 : -1;
            break;
        }
    const uint64_t *P = Aw, *Q = Bw;
    if (a.neg == b.neg) {
        uint64_t c = 0;
        for (int i = 0; i <= k; i++) {
            uint64_t s1 = Aw[i] + Bw[i];
            uint64_t c1 = s1 < Bw[i];
            uint64_t s2 = s1 + c;
            c = c1 | (s2 < c);
            S[i] = s2;
        }
        sign = a.neg;
    } else {
        if (cmp >= 0) {
            sign = a.neg;
        } else {
            P = Bw;
            Q = Aw;
            sign = b.neg;
        }
        uint64_t bw = 0;
        for (int i = 0; i <= k; i++) {
            uint64_t x = P[i], y = Q[i];
            S[i] = x - y - bw;
            bw = (x < y) || (x == y && bw);
        }
    }
    gf_normalize(res, sign, checked_add(win_bot, 64 * (k + 1), status), S, (int)k + 1, status);
    Mag rerr = gf_round(res, p, status);
    return units ? mag_add(rerr, mag_from_u64(units, win_bot)) : rerr;
}


}  // namespace apb
