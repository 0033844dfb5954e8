/* apb_oracle.c - TEST INFRASTRUCTURE ONLY (see apb_oracle.h).
 *
 * Plain-C restatement of the reference's ball dot product and block ball
 * matmul.  Paths below are relative to /root/reference/proj.  Compiled with
 * -ffp-contract=off so the binary64 radius sums round exactly like the
 * reference's x86-64 build (src/matmul.cpp:423-435, no FMA contraction).
 */
#include "apb_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;
typedef __int128 i128;

#define OL 200 /* max limbs of any temporary (p <= 8192 products) */

static int g_status;

/* --------------------------------------------------------------- Mag */
/* src/mag.cpp, include/apball/mag.hpp:15-59: (b/2^30)*2^f, 2^29 <= b < 2^30 */
enum { MZ = 0, MF = 1, MI = 2 };
typedef struct {
    int kind;
    uint64_t b;
    int64_t f;
} mag_t;

#define MAG_ONE (1ull << 30)
#define MEXP_MAX (INT64_MAX - 4)
#define MEXP_MIN (INT64_MIN + 4)

static mag_t mzero(void) { mag_t m = {MZ, 0, 0}; return m; }
static mag_t minf(void) { mag_t m = {MI, 0, 0}; return m; }

static unsigned bitw(uint64_t v) { return v ? 64u - (unsigned)__builtin_clzll(v) : 0u; }

/* Mag::from_parts (src/mag.cpp:18-31) */
static mag_t mparts(uint64_t b, int64_t f) {
    mag_t m;
    if (b == MAG_ONE) {
        b = MAG_ONE >> 1;
        if (f >= MEXP_MAX) return minf();
        f++;
    }
    m.kind = MF;
    m.b = b;
    m.f = f;
    return m;
}

/* Mag::from_u64_upper (src/mag.cpp:33-50) */
static mag_t mfrom_u64(uint64_t v, int64_t exp2) {
    if (v == 0) return mzero();
    unsigned len = bitw(v);
    uint64_t b;
    int inexact = 0;
    if (len <= 30) {
        b = v << (30 - len);
    } else {
        unsigned sh = len - 30;
        b = v >> sh;
        inexact = (v & ((1ull << sh) - 1)) != 0;
    }
    if (inexact) b++;
    i128 f = (i128)exp2 + len;
    if (f > MEXP_MAX) return minf();
    if (f < MEXP_MIN) return mparts(MAG_ONE >> 1, MEXP_MIN);
    return mparts(b, (int64_t)f);
}

/* Mag::from_double_upper (src/mag.cpp:79-87) */
static mag_t mfrom_double(double v, int64_t exp2) {
    if (v == 0.0) return mzero();
    if (isinf(v) || isnan(v)) return minf();
    int e;
    double fr = frexp(v, &e);
    uint64_t m53 = (uint64_t)ldexp(fr, 53);
    return mfrom_u64(m53, exp2 + e - 53);
}

/* mag_cmp (src/mag.cpp:99-106) */
static int mcmp(mag_t a, mag_t b) {
    int ra = a.kind == MZ ? 0 : (a.kind == MI ? 2 : 1);
    int rb = b.kind == MZ ? 0 : (b.kind == MI ? 2 : 1);
    if (ra != rb || ra != 1) return ra < rb ? -1 : (ra > rb ? 1 : 0);
    if (a.f != b.f) return a.f < b.f ? -1 : 1;
    if (a.b != b.b) return a.b < b.b ? -1 : 1;
    return 0;
}

/* mag_add_up (src/mag.cpp:108-130) */
static mag_t madd(mag_t a, mag_t b) {
    if (a.kind == MI || b.kind == MI) return minf();
    if (a.kind == MZ) return b;
    if (b.kind == MZ) return a;
    mag_t hi = a, lo = b;
    if (mcmp(hi, lo) < 0) {
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
    while (bh > MAG_ONE) {
        bh = (bh + 1) >> 1;
        if (f >= MEXP_MAX) return minf();
        f++;
    }
    return mparts(bh, f);
}

/* mag_mul_up (src/mag.cpp:132-145) */
static mag_t mmul(mag_t a, mag_t b) {
    if (a.kind == MZ || b.kind == MZ) return mzero();
    if (a.kind == MI || b.kind == MI) return minf();
    uint64_t p = a.b * b.b;
    uint64_t q = (p + (MAG_ONE - 1)) >> 30;
    i128 f = (i128)a.f + b.f;
    if (q < (MAG_ONE >> 1)) {
        q <<= 1;
        f--;
    }
    if (f > MEXP_MAX) return minf();
    if (f < MEXP_MIN) return mparts(MAG_ONE >> 1, MEXP_MIN);
    return mparts(q, (int64_t)f);
}

/* mag_ldexp (src/mag.cpp:166-172) */
static double mldexp(mag_t m, int64_t shift) {
    if (m.kind == MZ) return 0.0;
    return ldexp((double)m.b, (int)(m.f - 30 + shift));
}

/* ------------------------------------------------------------ ApFloat */
/* include/apball/apfloat.hpp:101-150; d[] little-endian, normalized */
typedef struct {
    int kind; /* APB_ZERO .. APB_NAN */
    int neg;
    int64_t e;
    int n;
    uint64_t d[OL];
} of_t;

#define EXP_HI (INT64_MAX - 8)
#define EXP_LO (INT64_MIN + 8)

static int64_t checked_exp(i128 e) {
    if (e > EXP_HI || e < EXP_LO) {
        g_status = APB_ERR_OVERFLOW;
        return 0;
    }
    return (int64_t)e;
}

static void ozero(of_t* x) {
    x->kind = APB_ZERO;
    x->neg = 0;
    x->e = 0;
    x->n = 0;
}

static int64_t obitwidth(const of_t* x) { return 64 * (int64_t)x->n - __builtin_ctzll(x->d[0]); }

/* apfloat_normalize (src/apfloat.cpp:116-136) */
static void onormalize(of_t* out, int neg, int64_t e, const uint64_t* raw, int nraw) {
    int h = nraw;
    while (h > 0 && raw[h - 1] == 0) h--;
    if (h == 0) {
        ozero(out);
        return;
    }
    unsigned tb = bitw(raw[h - 1]);
    i128 e_new = (i128)e - 64 * (int64_t)nraw + 64 * (int64_t)(h - 1) + tb;
    unsigned sh = (64 - tb) % 64;
    uint64_t m[OL];
    if (sh) {
        for (int i = h - 1; i > 0; i--) m[i] = (raw[i] << sh) | (raw[i - 1] >> (64 - sh));
        m[0] = raw[0] << sh;
    } else {
        memcpy(m, raw, sizeof(uint64_t) * (size_t)h);
    }
    int z = 0;
    while (m[z] == 0) z++;
    out->kind = APB_FINITE;
    out->neg = neg;
    out->e = checked_exp(e_new);
    out->n = h - z;
    memmove(out->d, m + z, sizeof(uint64_t) * (size_t)(h - z));
}

/* mag_upper_of_low_bits (src/apfloat.cpp:26-63) */
static mag_t mag_low_bits(const uint64_t* limbs, int cut_limbs, unsigned cut_bits, int64_t base) {
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
    if (t < 0) return mzero();
    unsigned tb = bitw(tv);
    uint64_t window = tb < 64 ? tv << (64 - tb) : tv;
    int low = 0;
    if (t > 0) {
        if (tb < 64) {
            window |= limbs[t - 1] >> tb;
            if (limbs[t - 1] & ((1ull << tb) - 1)) low = 1;
        } else if (limbs[t - 1]) {
            low = 1;
        }
        for (int i = 0; i + 1 < t && !low; i++)
            if (limbs[i]) low = 1;
    }
    uint64_t b = window >> 34;
    if (low || (window & ((1ull << 34) - 1))) b++;
    return mparts(b, checked_exp((i128)base + 64 * (int64_t)t + tb));
}

/* apfloat_round (src/apfloat.cpp:138-162): truncate toward zero */
static mag_t oround(of_t* x, int64_t p) {
    if (x->kind != APB_FINITE) return mzero();
    const int n = x->n;
    if (p >= 64 * (int64_t)n) return mzero();
    const int64_t cut = 64 * (int64_t)n - p;
    const int cut_limbs = (int)(cut / 64);
    const unsigned cut_bits = (unsigned)(cut % 64);
    mag_t err = mag_low_bits(x->d, cut_limbs, cut_bits, x->e - 64 * (int64_t)n);
    if (err.kind == MZ) return err;
    int keep = n - cut_limbs;
    uint64_t m[OL];
    memcpy(m, x->d + cut_limbs, sizeof(uint64_t) * (size_t)keep);
    if (cut_bits) m[0] &= ~((1ull << cut_bits) - 1);
    int z = 0;
    while (m[z] == 0) z++;
    x->n = keep - z;
    memcpy(x->d, m + z, sizeof(uint64_t) * (size_t)x->n);
    return err;
}

/* mul_limbs (include/apball/limb.hpp:137-143): schoolbook */
static void mul_limbs(const uint64_t* a, int na, const uint64_t* b, int nb, uint64_t* out) {
    memset(out, 0, sizeof(uint64_t) * (size_t)(na + nb));
    for (int j = 0; j < nb; j++) {
        uint64_t cy = 0;
        for (int i = 0; i < na; i++) {
            u128 t = (u128)a[i] * b[j] + cy + out[i + j];
            out[i + j] = (uint64_t)t;
            cy = (uint64_t)(t >> 64);
        }
        out[na + j] = cy;
    }
}

/* apfloat_mul_exact (src/apfloat.cpp:164-176) */
static void omul_exact(of_t* out, const of_t* a, const of_t* b) {
    if (a->kind == APB_NAN || b->kind == APB_NAN) {
        ozero(out);
        out->kind = APB_NAN;
        return;
    }
    int ainf = a->kind == APB_PINF || a->kind == APB_NINF;
    int binf = b->kind == APB_PINF || b->kind == APB_NINF;
    if (ainf || binf) {
        ozero(out);
        if (a->kind == APB_ZERO || b->kind == APB_ZERO) {
            out->kind = APB_NAN;
            return;
        }
        int sa = a->kind == APB_NINF || (a->kind == APB_FINITE && a->neg);
        int sb = b->kind == APB_NINF || (b->kind == APB_FINITE && b->neg);
        out->kind = (sa != sb) ? APB_NINF : APB_PINF;
        out->neg = sa != sb;
        return;
    }
    if (a->kind == APB_ZERO || b->kind == APB_ZERO) {
        ozero(out);
        return;
    }
    uint64_t prod[OL];
    mul_limbs(a->d, a->n, b->d, b->n, prod);
    onormalize(out, a->neg != b->neg, checked_exp((i128)a->e + b->e), prod, a->n + b->n);
}

/* place_truncated (src/apfloat.cpp:197-224) */
static int place_truncated(uint64_t* out, const of_t* x, int64_t win_bot) {
    const int n = x->n;
    const i128 off = (i128)x->e - 64 * (int64_t)n - win_bot;
    if (off >= 0) {
        int ol = (int)(off / 64);
        unsigned sh = (unsigned)(off % 64);
        for (int i = 0; i < n; i++) {
            out[ol + i] |= x->d[i] << sh;
            if (sh) out[ol + i + 1] |= x->d[i] >> (64 - sh);
        }
        return 0;
    }
    const i128 drop = -off;
    const i128 dl128 = drop / 64;
    const unsigned db = (unsigned)(drop % 64);
    if (dl128 >= n) return 1;
    const int dl = (int)dl128;
    int inexact = db && (x->d[dl] & ((1ull << db) - 1));
    for (int i = 0; i < dl && !inexact; i++)
        if (x->d[i]) inexact = 1;
    for (int i = dl; i < n; i++) {
        uint64_t v = db ? x->d[i] >> db : x->d[i];
        if (db && i + 1 < n) v |= x->d[i + 1] << (64 - db);
        out[i - dl] = v;
    }
    return inexact;
}

static int lcmp(const uint64_t* a, const uint64_t* b, int n) {
    for (int i = n - 1; i >= 0; i--)
        if (a[i] != b[i]) return a[i] > b[i] ? 1 : -1;
    return 0;
}
static void ladd(uint64_t* r, const uint64_t* a, const uint64_t* b, int n) {
    u128 c = 0;
    for (int i = 0; i < n; i++) {
        c += (u128)a[i] + b[i];
        r[i] = (uint64_t)c;
        c >>= 64;
    }
}
static void lsub(uint64_t* r, const uint64_t* a, const uint64_t* b, int n) {
    uint64_t bw = 0;
    for (int i = 0; i < n; i++) {
        uint64_t x = a[i], y = b[i];
        uint64_t d = x - y - bw;
        bw = (x < y) || (x == y && bw);
        r[i] = d;
    }
}

/* apfloat_add_round (src/apfloat.cpp:228-270) */
static mag_t oadd_round(of_t* res, const of_t* a, const of_t* b, int64_t p) {
    if (p < 2) p = 2;
    if (a->kind == APB_NAN || b->kind == APB_NAN) {
        ozero(res);
        res->kind = APB_NAN;
        return mzero();
    }
    int ainf = a->kind == APB_PINF || a->kind == APB_NINF;
    int binf = b->kind == APB_PINF || b->kind == APB_NINF;
    if (ainf || binf) {
        if (ainf && binf) {
            if (a->kind == b->kind) *res = *a;
            else {
                ozero(res);
                res->kind = APB_NAN;
            }
        } else {
            *res = ainf ? *a : *b;
        }
        return mzero();
    }
    if (a->kind == APB_ZERO) {
        *res = *b;
        return oround(res, p);
    }
    if (b->kind == APB_ZERO) {
        *res = *a;
        return oround(res, p);
    }
    const int64_t e_top = (a->e > b->e ? a->e : b->e) + 1;
    const i128 bot_a = (i128)a->e - 64 * (int64_t)a->n;
    const i128 bot_b = (i128)b->e - 64 * (int64_t)b->n;
    const i128 span = e_top - (bot_a < bot_b ? bot_a : bot_b);
    i128 k128 = (span + 63) / 64;
    const i128 budget = p / 64 + 3;
    if (k128 > budget) k128 = budget;
    const int k = (int)k128;
    const int64_t win_bot = checked_exp((i128)e_top - 64 * (int64_t)k);
    uint64_t A[OL], B[OL], S[OL];
    memset(A, 0, sizeof(uint64_t) * (size_t)(k + 1));
    memset(B, 0, sizeof(uint64_t) * (size_t)(k + 1));
    unsigned units = 0;
    units += (unsigned)place_truncated(A, a, win_bot);
    units += (unsigned)place_truncated(B, b, win_bot);
    int sign;
    if (a->neg == b->neg) {
        ladd(S, A, B, k + 1);
        sign = a->neg;
    } else if (lcmp(A, B, k + 1) >= 0) {
        lsub(S, A, B, k + 1);
        sign = a->neg;
    } else {
        lsub(S, B, A, k + 1);
        sign = b->neg;
    }
    onormalize(res, sign, checked_exp((i128)win_bot + 64 * (int64_t)(k + 1)), S, k + 1);
    mag_t rerr = oround(res, p);
    return units ? madd(rerr, mfrom_u64(units, win_bot)) : rerr;
}

/* mag_upper_from_apfloat (src/mag.cpp:147-153) */
static mag_t mupper(const of_t* x) {
    if (x->kind == APB_ZERO) return mzero();
    return mparts((x->d[x->n - 1] >> 34) + 1, x->e);
}

/* ------------------------------------------------------------ balls */
typedef struct {
    of_t m;
    mag_t r;
} ball_t;

static void load_of(of_t* x, const apb_balls* a, int64_t e) {
    uint8_t k = a->kind[e];
    ozero(x);
    x->kind = k & APB_KIND_MASK;
    x->neg = x->kind == APB_NINF;
    if (x->kind != APB_FINITE) return;
    const uint64_t* m = a->mant + e * (int64_t)a->L;
    int z = 0;
    while (z < a->L && m[z] == 0) z++;
    x->n = a->L - z;
    memcpy(x->d, m + z, sizeof(uint64_t) * (size_t)x->n);
    x->e = a->exp[e];
    x->neg = (k & APB_SIGN) != 0;
}

static mag_t load_mag(uint32_t b, int64_t f) {
    if (b == 0) return mzero();
    if (b == APB_RAD_INF) return minf();
    return mparts(b, f);
}

static void load_ball(ball_t* b, const apb_balls* a, int64_t e) {
    load_of(&b->m, a, e);
    b->r = load_mag(a->rad_man[e], a->rad_exp[e]);
}

static void store_ball(apb_balls* a, int64_t e, const of_t* m, mag_t r) {
    uint64_t* dst = a->mant + e * (int64_t)a->L;
    memset(dst, 0, sizeof(uint64_t) * (size_t)a->L);
    a->exp[e] = 0;
    a->kind[e] = (uint8_t)m->kind;
    if (m->kind == APB_FINITE) {
        if (m->n > a->L) g_status = APB_ERR_UNSUPPORTED;
        else memcpy(dst + (a->L - m->n), m->d, sizeof(uint64_t) * (size_t)m->n);
        a->exp[e] = m->e;
        if (m->neg) a->kind[e] |= APB_SIGN;
    }
    if (r.kind == MZ) {
        a->rad_man[e] = 0;
        a->rad_exp[e] = 0;
    } else if (r.kind == MI) {
        a->rad_man[e] = APB_RAD_INF;
        a->rad_exp[e] = 0;
    } else {
        a->rad_man[e] = (uint32_t)r.b;
        a->rad_exp[e] = r.f;
    }
}

static int ofinite(const of_t* x) { return x->kind == APB_ZERO || x->kind == APB_FINITE; }

static void oneg(of_t* x) {
    if (x->kind == APB_FINITE) x->neg = !x->neg;
    else if (x->kind == APB_PINF) {
        x->kind = APB_NINF;
        x->neg = 1;
    } else if (x->kind == APB_NINF) {
        x->kind = APB_PINF;
        x->neg = 0;
    }
}

static void set_indeterminate(ball_t* r) {
    ozero(&r->m);
    r->m.kind = APB_NAN;
    r->r = minf();
}

/* ball_fallback_addmul (src/ball.cpp:21-36) */
static void ball_addmul(ball_t* acc, const ball_t* x, const ball_t* y, int64_t p) {
    if (acc->m.kind == APB_NAN || x->m.kind == APB_NAN || y->m.kind == APB_NAN) {
        set_indeterminate(acc);
        return;
    }
    static of_t prod, mid;
    omul_exact(&prod, &x->m, &y->m);
    if (prod.kind == APB_NAN) {
        set_indeterminate(acc);
        return;
    }
    mag_t rad = acc->r;
    if (y->r.kind != MZ && x->m.kind != APB_ZERO) rad = madd(rad, mmul(mupper(&x->m), y->r));
    if (x->r.kind != MZ && y->m.kind != APB_ZERO) rad = madd(rad, mmul(mupper(&y->m), x->r));
    if (x->r.kind != MZ && y->r.kind != MZ) rad = madd(rad, mmul(x->r, y->r));
    mag_t perr = oround(&prod, p);
    mag_t aerr = oadd_round(&mid, &acc->m, &prod, p);
    if (mid.kind == APB_NAN) {
        set_indeterminate(acc);
        return;
    }
    acc->m = mid;
    acc->r = madd(rad, madd(perr, aerr));
}

/* ball_add (src/ball.cpp:15-19) */
static void ball_add(ball_t* res, const ball_t* a, const ball_t* b, int64_t p) {
    static of_t mid;
    mag_t err = oadd_round(&mid, &a->m, &b->m, p);
    if (mid.kind == APB_NAN) {
        set_indeterminate(res);
        return;
    }
    mag_t r = madd(madd(a->r, b->r), err);
    res->m = mid;
    res->r = r;
}

/* ------------------------------------------------------------ dot */
/* DotPlan (include/apball/dot.hpp:25-36), setup_core (src/dot.cpp:72-134) */
enum { ST_PROCEED = 0, ST_FALLBACK = 1, ST_ZERO = 2 };
typedef struct {
    int64_t e_max, e_min, e_rad;
    uint64_t nnz;
    int64_t p_eff;
    unsigned extend, padding;
    int n_s;
    int64_t e_s;
    int status;
} plan_t;

typedef struct {
    const ball_t* x;
    const ball_t* y;
    int neg;
} term_t;

#define EXP_CAP (1ll << 60)
static int huge(int64_t e) { return e > EXP_CAP || e < -EXP_CAP; }

static int g_disable_reduction;

static plan_t setup(const term_t* t, int64_t total, int64_t p, int with_radius) {
    plan_t pl;
    pl.e_max = INT64_MIN;
    pl.e_min = INT64_MAX;
    pl.e_rad = INT64_MIN;
    pl.nnz = 0;
    pl.p_eff = 2;
    pl.extend = pl.padding = 0;
    pl.n_s = 0;
    pl.e_s = 0;
    pl.status = ST_ZERO;
    const int track_min = p > 128;
    for (int64_t i = 0; i < total; i++) {
        const of_t* xm = &t[i].x->m;
        const of_t* ym = &t[i].y->m;
        if (!ofinite(xm) || !ofinite(ym)) {
            pl.status = ST_FALLBACK;
            return pl;
        }
        if ((xm->kind != APB_ZERO && huge(xm->e)) || (ym->kind != APB_ZERO && huge(ym->e))) {
            pl.status = ST_FALLBACK;
            return pl;
        }
        if (xm->kind != APB_ZERO && ym->kind != APB_ZERO) {
            pl.nnz++;
            int64_t ee = xm->e + ym->e;
            if (ee > pl.e_max) pl.e_max = ee;
            if (track_min) {
                int64_t lo = ee - 64 * (int64_t)(xm->n + ym->n);
                if (lo < pl.e_min) pl.e_min = lo;
            }
        }
        if (with_radius) {
            mag_t xr = t[i].x->r, yr = t[i].y->r;
            if (xr.kind == MI || yr.kind == MI || (xr.kind != MZ && huge(xr.f)) ||
                (yr.kind != MZ && huge(yr.f))) {
                pl.status = ST_FALLBACK;
                return pl;
            }
            if (yr.kind != MZ && xm->kind != APB_ZERO && xm->e + yr.f > pl.e_rad) pl.e_rad = xm->e + yr.f;
            if (xr.kind != MZ && ym->kind != APB_ZERO && ym->e + xr.f > pl.e_rad) pl.e_rad = ym->e + xr.f;
            if (xr.kind != MZ && yr.kind != MZ && xr.f + yr.f > pl.e_rad) pl.e_rad = xr.f + yr.f;
        }
    }
    if (pl.e_max == INT64_MIN && pl.e_rad == INT64_MIN) {
        pl.status = ST_ZERO;
        return pl;
    }
    if (pl.e_max == INT64_MIN) {
        p = 2;
    } else if (!g_disable_reduction) {
        if (pl.e_rad != INT64_MIN && pl.e_max - pl.e_rad + 30 < p) p = pl.e_max - pl.e_rad + 30;
        if (pl.e_min != INT64_MAX && pl.e_max - pl.e_min + 30 < p) p = pl.e_max - pl.e_min + 30;
        if (p < 2) p = 2;
    }
    pl.p_eff = p;
    pl.padding = 4 + bitw((uint64_t)total);
    pl.extend = bitw(pl.nnz) + 1;
    int64_t ns = (p + pl.extend + pl.padding + 63) / 64;
    pl.n_s = (int)(ns < 2 ? 2 : ns);
    pl.e_s = pl.e_max == INT64_MIN ? 0 : pl.e_max + pl.extend;
    pl.status = ST_PROCEED;
    return pl;
}

typedef struct {
    uint64_t s[OL];
    uint64_t err;
    uint64_t srad;
} acc_t;

/* mulhigh_approx (include/apball/limb.hpp:194-228) */
static void mulhigh(const uint64_t* a, int na, const uint64_t* b, int nb, int k, uint64_t* out) {
    const int total = na + nb;
    if (k == total) {
        mul_limbs(a, na, b, nb, out);
        return;
    }
    const int base = total - k >= 2 ? total - k - 2 : 0;
    const int wlen = total - base;
    uint64_t w[2 * OL];
    memset(w, 0, sizeof(uint64_t) * (size_t)wlen);
    for (int j = 0; j < nb; j++) {
        int i0 = base > j ? base - j : 0;
        if (i0 >= na) continue;
        int len = na - i0;
        int off = i0 + j - base;
        uint64_t cy = 0;
        for (int i = 0; i < len; i++) {
            u128 t = (u128)a[i0 + i] * b[j] + cy + w[off + i];
            w[off + i] = (uint64_t)t;
            cy = (uint64_t)(t >> 64);
        }
        for (int q = off + len; q < wlen && cy; q++) {
            uint64_t s = w[q] + cy;
            cy = s < cy;
            w[q] = s;
        }
    }
    memcpy(out, w + (wlen - k), sizeof(uint64_t) * (size_t)k);
}

/* accumulate_aligned (src/dot.cpp:139-173) */
static void acc_aligned(const plan_t* pl, acc_t* acc, const uint64_t* t, int nt, int64_t e_term,
                        int negate) {
    const int64_t shift = pl->e_s - e_term;
    if (shift >= 64 * (int64_t)pl->n_s) {
        acc->err++;
        return;
    }
    const unsigned sb = (unsigned)(shift % 64);
    const int sl = (int)(shift / 64);
    uint64_t buf[OL];
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
    const int avail = pl->n_s - sl;
    int ds, dt, v;
    if (nt <= avail) {
        ds = avail - nt;
        dt = 0;
        v = nt;
    } else {
        ds = 0;
        dt = nt - avail;
        v = avail;
        acc->err++;
    }
    /* add_signed_range (include/apball/limb.hpp:149-169), wrapping at the top */
    uint64_t* w = acc->s + ds;
    if (!negate) {
        u128 c = 0;
        for (int i = 0; i < v; i++) {
            c += (u128)w[i] + t[dt + i];
            w[i] = (uint64_t)c;
            c >>= 64;
        }
        for (int i = v; ds + i < pl->n_s && c; i++) {
            c += w[i];
            w[i] = (uint64_t)c;
            c >>= 64;
        }
    } else {
        uint64_t bw = 0;
        for (int i = 0; i < v; i++) {
            uint64_t x = w[i], y = t[dt + i];
            uint64_t d = x - y - bw;
            bw = (x < y) || (x == y && bw);
            w[i] = d;
        }
        for (int i = v; ds + i < pl->n_s && bw; i++) {
            uint64_t x = w[i];
            w[i] = x - 1;
            bw = x == 0;
        }
    }
}

/* dot_accumulate_term general path (src/dot.cpp:229-273); the inline
 * 2x2 path (:241-247) is bit-identical to it (tests/test_dot.cpp:170-189). */
static void acc_term(const plan_t* pl, acc_t* acc, const of_t* m, const of_t* mp, int negate) {
    negate ^= m->neg ^ mp->neg;
    const int64_t e_term = m->e + mp->e;
    const int64_t shift = pl->e_s - e_term;
    if (shift >= 64 * (int64_t)pl->n_s) {
        acc->err++;
        return;
    }
    const int n = m->n, np = mp->n;
    const int64_t p_t = 64 * (int64_t)pl->n_s - shift;
    const int ncap = (int)((p_t + 63) / 64) + 1;
    const int na = n < ncap ? n : ncap, nb = np < ncap ? np : ncap;
    if (n > ncap || np > ncap) acc->err++;
    const uint64_t* a = m->d + (n - na);
    const uint64_t* b = mp->d + (np - nb);
    const int nt = na + nb;
    uint64_t t[2 * OL];
    int lead = nt;
    int short_prod = 0;
    const int mn = n < np ? n : np;
    if (p_t >= 25 * 64 && 640 * (int64_t)mn > 9 * p_t) {
        const int v = pl->n_s - (int)(shift / 64);
        const int k = nt < v + 1 ? nt : v + 1;
        if (k < nt) {
            mulhigh(a, na, b, nb, k, t);
            acc->err++;
            lead = k;
            short_prod = 1;
        }
    }
    if (!short_prod) mul_limbs(a, na, b, nb, t);
    acc_aligned(pl, acc, t, lead, e_term, negate);
}

/* srad_add / radius_pass_term (src/dot.cpp:282-295, 346-358) */
static void srad_add(uint64_t* srad, uint64_t ab, int64_t af, uint64_t bb, int64_t bf,
                     int64_t e_rad) {
    int64_t d = e_rad - (af + bf);
    if (d < 30) *srad += ((ab * bb) >> (30 + d)) + 1;
    else *srad += 1;
}

static void rad_term(const plan_t* pl, acc_t* acc, const term_t* t) {
    const of_t* xm = &t->x->m;
    const of_t* ym = &t->y->m;
    mag_t xr = t->x->r, yr = t->y->r;
    if (yr.kind != MZ && xm->kind != APB_ZERO)
        srad_add(&acc->srad, (xm->d[xm->n - 1] >> 34) + 1, xm->e, yr.b, yr.f, pl->e_rad);
    if (xr.kind != MZ && ym->kind != APB_ZERO)
        srad_add(&acc->srad, (ym->d[ym->n - 1] >> 34) + 1, ym->e, xr.b, xr.f, pl->e_rad);
    if (xr.kind != MZ && yr.kind != MZ) srad_add(&acc->srad, xr.b, xr.f, yr.b, yr.f, pl->e_rad);
}

/* dot_finalize (src/dot.cpp:306-321) */
static void finalize(const plan_t* pl, acc_t* acc, int64_t p, of_t* mid, mag_t* rad, int with_radius) {
    if (p > pl->p_eff) p = pl->p_eff;
    if (p < 2) p = 2;
    int sign = 0;
    uint64_t s[OL];
    memcpy(s, acc->s, sizeof(uint64_t) * (size_t)pl->n_s);
    if (s[pl->n_s - 1] >> 63) {
        /* neg_in_place (include/apball/limb.hpp:180-187) */
        int i = 0;
        while (i < pl->n_s && s[i] == 0) i++;
        if (i < pl->n_s) {
            s[i] = ~s[i] + 1;
            for (i++; i < pl->n_s; i++) s[i] = ~s[i];
        }
        sign = 1;
    }
    onormalize(mid, sign, pl->e_s, s, pl->n_s);
    mag_t r = oround(mid, p);
    if (with_radius) {
        if (acc->err) r = madd(r, mfrom_u64(acc->err, pl->e_s - 64 * (int64_t)pl->n_s));
        if (acc->srad) r = madd(r, mfrom_u64(acc->srad, pl->e_rad - 30));
    } else {
        r = mzero(); /* dot_approx_core returns the midpoint only (src/dot.cpp:377-400) */
    }
    *rad = r;
}

static ball_t g_one;
static void init_one(void) {
    uint64_t l = 1ull << 63;
    onormalize(&g_one.m, 0, 1, &l, 1);
    g_one.r = mzero();
}

static int64_t xel(const apb_dot_index* ix, int64_t b, int64_t i) {
    return ix->x_off + (b / ix->bdiv) * ix->xs1 + (b % ix->bdiv) * ix->xs2 + i * ix->xstep;
}
static int64_t yel(const apb_dot_index* ix, int64_t b, int64_t i) {
    return ix->y_off + (b / ix->bdiv) * ix->ys1 + (b % ix->bdiv) * ix->ys2 + i * ix->ystep;
}

/* dot_ball_core / dot_approx_core over a term list (src/dot.cpp:361-400) */
static void dot_core(const term_t* terms, int64_t total, int64_t p, int approx, of_t* mid,
                     mag_t* rad, apb_dot_state* st, uint64_t* accout, int64_t acc_stride) {
    plan_t pl = setup(terms, total, p, !approx);
    if (st) {
        memset(st, 0, sizeof *st);
        st->e_max = pl.e_max;
        st->e_min = pl.e_min;
        st->e_rad = pl.e_rad;
        st->n_nonzero = pl.nnz;
        st->p_eff = pl.p_eff;
        st->extend = (int32_t)pl.extend;
        st->padding = (int32_t)pl.padding;
        st->n_s = pl.n_s;
        st->e_s = pl.e_s;
        st->status = pl.status;
    }
    if (pl.status == ST_ZERO) {
        ozero(mid);
        *rad = mzero();
        return;
    }
    if (pl.status == ST_FALLBACK) {
        /* fallback_ball / fallback_approx (src/dot.cpp:325-344) */
        static ball_t acc, yy;
        ozero(&acc.m);
        acc.r = mzero();
        for (int64_t i = 0; i < total; i++) {
            yy = *terms[i].y;
            if (terms[i].neg) oneg(&yy.m);
            if (approx) {
                static of_t prod, s;
                omul_exact(&prod, &terms[i].x->m, &yy.m);
                oround(&prod, p);
                oadd_round(&s, &acc.m, &prod, p);
                acc.m = s;
            } else {
                ball_addmul(&acc, terms[i].x, &yy, p);
            }
        }
        *mid = acc.m;
        *rad = approx ? mzero() : acc.r;
        return;
    }
    static acc_t acc;
    memset(acc.s, 0, sizeof(uint64_t) * (size_t)pl.n_s);
    acc.err = 0;
    acc.srad = 0;
    for (int64_t i = 0; i < total; i++) {
        const term_t* t = &terms[i];
        if (t->x->m.kind != APB_ZERO && t->y->m.kind != APB_ZERO)
            acc_term(&pl, &acc, &t->x->m, &t->y->m, t->neg);
        if (!approx) rad_term(&pl, &acc, t);
    }
    if (st) {
        st->err = acc.err;
        st->srad = acc.srad;
    }
    if (accout)
        for (int l = 0; l < pl.n_s && l < acc_stride; l++) accout[l] = acc.s[l];
    finalize(&pl, &acc, p, mid, rad, !approx);
}

int orc_dot_batch(const apb_balls* x, const apb_balls* y, const apb_balls* initial, int subtract,
                  const apb_dot_index* idx, int64_t n, int64_t batch, int64_t prec, int mode,
                  int disable_reduction, apb_balls* out, apb_dot_state* state, uint64_t* acc,
                  int64_t acc_stride) {
    g_status = APB_OK;
    g_disable_reduction = disable_reduction;
    init_one();
    ball_t* xs = (ball_t*)malloc(sizeof(ball_t) * (size_t)(n + 1));
    ball_t* ys = (ball_t*)malloc(sizeof(ball_t) * (size_t)(n + 1));
    term_t* terms = (term_t*)malloc(sizeof(term_t) * (size_t)(n + 1));
    static of_t mid;
    for (int64_t b = 0; b < batch; b++) {
        for (int64_t i = 0; i < n; i++) {
            load_ball(&xs[i], x, xel(idx, b, i));
            load_ball(&ys[i], y, yel(idx, b, i));
            terms[i].x = &xs[i];
            terms[i].y = &ys[i];
            terms[i].neg = subtract != 0;
        }
        int64_t total = n;
        if (initial) {
            load_ball(&xs[n], initial, b);
            terms[n].x = &xs[n];
            terms[n].y = &g_one;
            terms[n].neg = 0;
            total++;
        }
        mag_t rad;
        dot_core(terms, total, prec, mode == APB_DOT_APPROX, &mid, &rad, state ? &state[b] : NULL,
                 acc ? acc + b * acc_stride : NULL, acc_stride);
        store_ball(out, b, &mid, rad);
    }
    free(xs);
    free(ys);
    free(terms);
    g_disable_reduction = 0;
    return g_status;
}

int orc_dot_complex_batch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                          const apb_balls* yim, const apb_dot_index* idx, int64_t n,
                          int64_t batch, int64_t prec, int mode, apb_balls* ore, apb_balls* oim) {
    g_status = APB_OK;
    const int approx = mode == APB_DOT_APPROX;
    ball_t* u = (ball_t*)malloc(sizeof(ball_t) * (size_t)(2 * n + 1));
    ball_t* v = (ball_t*)malloc(sizeof(ball_t) * (size_t)(2 * n + 1));
    term_t* tre = (term_t*)malloc(sizeof(term_t) * (size_t)(2 * n + 1));
    term_t* tim = (term_t*)malloc(sizeof(term_t) * (size_t)(2 * n + 1));
    static of_t mre, mim;
    for (int64_t b = 0; b < batch; b++) {
        for (int64_t j = 0; j < n; j++) {
            int64_t ex = xel(idx, b, j), ey = yel(idx, b, j);
            load_ball(&u[2 * j], xre, ex);
            load_ball(&u[2 * j + 1], xim, ex);
            load_ball(&v[2 * j], yre, ey);
            load_ball(&v[2 * j + 1], yim, ey);
            /* ComplexPartView (src/dot.cpp:52-68): re = ac - bd, im = ad + bc */
            tre[2 * j] = (term_t){&u[2 * j], &v[2 * j], 0};
            tre[2 * j + 1] = (term_t){&u[2 * j + 1], &v[2 * j + 1], 1};
            tim[2 * j] = (term_t){&u[2 * j], &v[2 * j + 1], 0};
            tim[2 * j + 1] = (term_t){&u[2 * j + 1], &v[2 * j], 0};
        }
        plan_t pre = setup(tre, 2 * n, prec, !approx);
        plan_t pim = setup(tim, 2 * n, prec, !approx);
        mag_t rre = mzero(), rim = mzero();
        if (pre.status == ST_FALLBACK || pim.status == ST_FALLBACK) {
            /* complex_fallback_ball (src/dot.cpp:532-545) */
            static ball_t are, aim, nb;
            ozero(&are.m);
            are.r = mzero();
            ozero(&aim.m);
            aim.r = mzero();
            for (int64_t j = 0; j < n; j++) {
                ball_addmul(&are, &u[2 * j], &v[2 * j], prec);
                nb = v[2 * j + 1];
                oneg(&nb.m);
                ball_addmul(&are, &u[2 * j + 1], &nb, prec);
                ball_addmul(&aim, &u[2 * j], &v[2 * j + 1], prec);
                ball_addmul(&aim, &u[2 * j + 1], &v[2 * j], prec);
            }
            mre = are.m;
            mim = aim.m;
            rre = approx ? mzero() : are.r;
            rim = approx ? mzero() : aim.r;
        } else {
            dot_core(tre, 2 * n, prec, approx, &mre, &rre, NULL, NULL, 0);
            dot_core(tim, 2 * n, prec, approx, &mim, &rim, NULL, NULL, 0);
        }
        store_ball(ore, b, &mre, rre);
        store_ball(oim, b, &mim, rim);
    }
    free(u);
    free(v);
    free(tre);
    free(tim);
    return g_status;
}

/* ------------------------------------------------------------ matmul */

static void mat_load(ball_t* dst, const apb_mat* m) {
    for (int64_t i = 0; i < m->rows * m->cols; i++) load_ball(&dst[i], &m->b, i);
}

/* entry_precision (src/matmul.cpp:47-52) */
static int64_t entry_precision(const ball_t* m, int64_t cnt) {
    int64_t p = 0;
    for (int64_t i = 0; i < cnt; i++)
        if (m[i].m.kind == APB_FINITE && obitwidth(&m[i].m) > p) p = obitwidth(&m[i].m);
    return p;
}

typedef struct {
    int64_t top, bot;
} win_t;

/* greedy_split (src/matmul.cpp:74-114) over precomputed entry windows:
 * wa[i*n+k] for A rows, wb[j*n+k] for B columns; valid iff top != INT64_MIN */
static int64_t greedy_split(int64_t n, int64_t mr, int64_t kc, const win_t* ea, const win_t* eb,
                            int64_t h, int64_t* out) {
    win_t* wa = (win_t*)malloc(sizeof(win_t) * (size_t)(mr ? mr : 1));
    win_t* wb = (win_t*)malloc(sizeof(win_t) * (size_t)(kc ? kc : 1));
    int64_t cnt = 0, lo = 0, k = 0;
#define RESET()                                                            \
    do {                                                                   \
        for (int64_t q = 0; q < mr; q++) wa[q] = (win_t){INT64_MIN, INT64_MAX}; \
        for (int64_t q = 0; q < kc; q++) wb[q] = (win_t){INT64_MIN, INT64_MAX}; \
    } while (0)
    RESET();
    while (lo < n) {
        int ok = k == lo;
        if (!ok) {
            ok = 1;
            for (int64_t i = 0; i < mr && ok; i++) {
                win_t e = ea[i * n + k];
                if (e.top == INT64_MIN) continue;
                int64_t w = wa[i].top == INT64_MIN
                                ? e.top - e.bot
                                : (wa[i].top > e.top ? wa[i].top : e.top) - (wa[i].bot < e.bot ? wa[i].bot : e.bot);
                if (w > h) ok = 0;
            }
            for (int64_t j = 0; j < kc && ok; j++) {
                win_t e = eb[j * n + k];
                if (e.top == INT64_MIN) continue;
                int64_t w = wb[j].top == INT64_MIN
                                ? e.top - e.bot
                                : (wb[j].top > e.top ? wb[j].top : e.top) - (wb[j].bot < e.bot ? wb[j].bot : e.bot);
                if (w > h) ok = 0;
            }
        }
        if (ok) {
            for (int64_t i = 0; i < mr; i++) {
                win_t e = ea[i * n + k];
                if (e.top == INT64_MIN) continue;
                if (e.top > wa[i].top) wa[i].top = e.top;
                if (e.bot < wa[i].bot) wa[i].bot = e.bot;
            }
            for (int64_t j = 0; j < kc; j++) {
                win_t e = eb[j * n + k];
                if (e.top == INT64_MIN) continue;
                if (e.top > wb[j].top) wb[j].top = e.top;
                if (e.bot < wb[j].bot) wb[j].bot = e.bot;
            }
            if (++k == n) {
                out[2 * cnt] = lo;
                out[2 * cnt + 1] = k;
                cnt++;
                lo = k;
            }
        } else {
            out[2 * cnt] = lo;
            out[2 * cnt + 1] = k;
            cnt++;
            lo = k;
            RESET();
        }
    }
#undef RESET
    free(wa);
    free(wb);
    return cnt;
}

static win_t ball_window(const ball_t* e) {
    win_t w = {INT64_MIN, INT64_MAX};
    if (e->m.kind != APB_FINITE) return w;
    w.top = e->m.e;
    w.bot = e->m.e - obitwidth(&e->m);
    return w;
}

/* plan_blocks (src/matmul.cpp:132-161) */
static int64_t plan_blocks(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N,
                           int64_t p, int64_t* steps) {
    if (K == 0) return 0;
    int64_t pa = entry_precision(a, M * K), pb = entry_precision(b, K * N);
    int64_t pm = pa > pb ? pa : pb;
    if (p < pm) pm = p;
    const int64_t h = (5 * pm) / 4 + 192;
    win_t* ea = (win_t*)malloc(sizeof(win_t) * (size_t)(M * K));
    win_t* eb = (win_t*)malloc(sizeof(win_t) * (size_t)(N * K));
    for (int64_t i = 0; i < M; i++)
        for (int64_t k = 0; k < K; k++) ea[i * K + k] = ball_window(&a[i * K + k]);
    for (int64_t j = 0; j < N; j++)
        for (int64_t k = 0; k < K; k++) eb[j * K + k] = ball_window(&b[k * N + j]);
    int64_t* raw = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * K + 2));
    int64_t nraw = greedy_split(K, M, N, ea, eb, h, raw);
    int64_t ns = 0;
    for (int64_t idx = 0; idx < nraw; idx++) {
        int64_t lo = raw[2 * idx], hi = raw[2 * idx + 1];
        if (hi - lo < 30) {
            hi = lo + 30 < K ? lo + 30 : K;
            while (idx + 1 < nraw && raw[2 * (idx + 1) + 1] <= hi) idx++;
            if (idx + 1 < nraw && raw[2 * (idx + 1)] < hi) raw[2 * (idx + 1)] = hi;
            steps[3 * ns] = lo;
            steps[3 * ns + 1] = hi;
            steps[3 * ns + 2] = 1;
        } else {
            steps[3 * ns] = lo;
            steps[3 * ns + 1] = hi;
            steps[3 * ns + 2] = 0;
        }
        ns++;
    }
    free(raw);
    free(ea);
    free(eb);
    return ns;
}

int orc_plan_blocks(const apb_mat* A, const apb_mat* B, int64_t prec, int64_t* steps,
                    int64_t max_steps, int64_t* n_steps) {
    g_status = APB_OK;
    if (A->cols != B->rows) return APB_ERR_INVALID;
    ball_t* a = (ball_t*)malloc(sizeof(ball_t) * (size_t)(A->rows * A->cols + 1));
    ball_t* b = (ball_t*)malloc(sizeof(ball_t) * (size_t)(B->rows * B->cols + 1));
    mat_load(a, A);
    mat_load(b, B);
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(3 * A->cols + 3));
    int64_t ns = plan_blocks(a, A->rows, A->cols, b, B->cols, prec, tmp);
    *n_steps = ns;
    for (int64_t i = 0; i < ns && i < max_steps; i++)
        for (int q = 0; q < 3; q++) steps[3 * i + q] = tmp[3 * i + q];
    free(tmp);
    free(a);
    free(b);
    return g_status;
}

/* Scaled integers (scale_block_rows/cols, src/matmul.cpp:163-203;
 * bigint_from_apfloat_scaled, src/bigint.cpp:178-185) kept as W-limb two's
 * complement words; products summed in W2-limb two's complement. */
static void to_scaled(uint64_t* dst, int W, const of_t* x, int64_t shift) {
    memset(dst, 0, sizeof(uint64_t) * (size_t)W);
    if (x->kind != APB_FINITE) return;
    int64_t sh = x->e - 64 * (int64_t)x->n + shift; /* value = mant * 2^sh, sh may be < 0 */
    /* mant has low-limb trailing zeros >= -sh (exactness, scale_block_*) */
    uint64_t tmp[OL + 2];
    memset(tmp, 0, sizeof tmp);
    if (sh >= 0) {
        int wl = (int)(sh / 64);
        unsigned bb = (unsigned)(sh % 64);
        for (int i = 0; i < x->n; i++) {
            tmp[wl + i] |= x->d[i] << bb;
            if (bb) tmp[wl + i + 1] |= x->d[i] >> (64 - bb);
        }
    } else {
        int64_t r = -sh;
        int wl = (int)(r / 64);
        unsigned bb = (unsigned)(r % 64);
        for (int i = wl; i < x->n; i++) {
            uint64_t v = bb ? x->d[i] >> bb : x->d[i];
            if (bb && i + 1 < x->n) v |= x->d[i + 1] << (64 - bb);
            tmp[i - wl] = v;
        }
    }
    memcpy(dst, tmp, sizeof(uint64_t) * (size_t)W);
    if (x->neg) {
        uint64_t c = 1;
        for (int i = 0; i < W; i++) {
            uint64_t v = ~dst[i] + c;
            c = (c && v == 0);
            dst[i] = v;
        }
    }
}

/* T[i,j] = sum_k a[i,k] b[k,j], exact two's complement (int_matmul, src/matmul.cpp:264-364) */
static void int_gemm(const uint64_t* ia, const uint64_t* ib, int64_t M, int64_t K, int64_t N, int W,
                     uint64_t* T, int W2) {
    memset(T, 0, sizeof(uint64_t) * (size_t)(M * N * W2));
    uint64_t pa[OL], pb[OL], pr[2 * OL];
    for (int64_t i = 0; i < M; i++)
        for (int64_t j = 0; j < N; j++) {
            uint64_t* acc = T + (i * N + j) * W2;
            for (int64_t k = 0; k < K; k++) {
                const uint64_t* x = ia + (i * K + k) * W;
                const uint64_t* y = ib + (k * N + j) * W;
                int nx = x[W - 1] >> 63, ny = y[W - 1] >> 63;
                memcpy(pa, x, sizeof(uint64_t) * (size_t)W);
                memcpy(pb, y, sizeof(uint64_t) * (size_t)W);
                if (nx) {
                    uint64_t c = 1;
                    for (int q = 0; q < W; q++) {
                        uint64_t v = ~pa[q] + c;
                        c = (c && v == 0);
                        pa[q] = v;
                    }
                }
                if (ny) {
                    uint64_t c = 1;
                    for (int q = 0; q < W; q++) {
                        uint64_t v = ~pb[q] + c;
                        c = (c && v == 0);
                        pb[q] = v;
                    }
                }
                int zx = 1, zy = 1;
                for (int q = 0; q < W; q++) {
                    if (pa[q]) zx = 0;
                    if (pb[q]) zy = 0;
                }
                if (zx || zy) continue;
                mul_limbs(pa, W, pb, W, pr);
                for (int q = 2 * W; q < W2; q++) pr[q] = 0;
                if (nx != ny) {
                    uint64_t bw = 0;
                    for (int q = 0; q < W2; q++) {
                        uint64_t a0 = acc[q], b0 = pr[q];
                        uint64_t d = a0 - b0 - bw;
                        bw = (a0 < b0) || (a0 == b0 && bw);
                        acc[q] = d;
                    }
                } else {
                    u128 c = 0;
                    for (int q = 0; q < W2; q++) {
                        c += (u128)acc[q] + pr[q];
                        acc[q] = (uint64_t)c;
                        c >>= 64;
                    }
                }
            }
        }
}

static void scale_block(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N,
                        int64_t lo, int64_t hi, int64_t* ei, int64_t* fj, int W, uint64_t* ia,
                        uint64_t* ib) {
    const int64_t w = hi - lo;
    for (int64_t i = 0; i < M; i++) {
        int64_t bot = INT64_MAX;
        for (int64_t k = lo; k < hi; k++) {
            const of_t* e = &a[i * K + k].m;
            if (e->kind != APB_ZERO && e->e - obitwidth(e) < bot) bot = e->e - obitwidth(e);
        }
        ei[i] = bot == INT64_MAX ? 0 : -bot;
        for (int64_t k = lo; k < hi; k++) to_scaled(ia + (i * w + (k - lo)) * W, W, &a[i * K + k].m, ei[i]);
    }
    for (int64_t j = 0; j < N; j++) {
        int64_t bot = INT64_MAX;
        for (int64_t k = lo; k < hi; k++) {
            const of_t* e = &b[k * N + j].m;
            if (e->kind != APB_ZERO && e->e - obitwidth(e) < bot) bot = e->e - obitwidth(e);
        }
        fj[j] = bot == INT64_MAX ? 0 : -bot;
        for (int64_t k = lo; k < hi; k++) to_scaled(ib + ((k - lo) * N + j) * W, W, &b[k * N + j].m, fj[j]);
    }
}

static int block_width(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N,
                       int64_t lo, int64_t hi) {
    /* limbs for the largest scaled entry plus a sign bit */
    int64_t h = 0;
    for (int64_t i = 0; i < M; i++) {
        int64_t top = INT64_MIN, bot = INT64_MAX;
        for (int64_t k = lo; k < hi; k++) {
            const of_t* e = &a[i * K + k].m;
            if (e->kind != APB_FINITE) continue;
            if (e->e > top) top = e->e;
            if (e->e - obitwidth(e) < bot) bot = e->e - obitwidth(e);
        }
        if (top != INT64_MIN && top - bot > h) h = top - bot;
    }
    for (int64_t j = 0; j < N; j++) {
        int64_t top = INT64_MIN, bot = INT64_MAX;
        for (int64_t k = lo; k < hi; k++) {
            const of_t* e = &b[k * N + j].m;
            if (e->kind != APB_FINITE) continue;
            if (e->e > top) top = e->e;
            if (e->e - obitwidth(e) < bot) bot = e->e - obitwidth(e);
        }
        if (top != INT64_MIN && top - bot > h) h = top - bot;
    }
    return (int)((h + 1 + 63) / 64);
}

int orc_block_int_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi,
                          int64_t* row_scale, int64_t* col_scale, uint64_t* out,
                          int64_t out_limbs) {
    g_status = APB_OK;
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    ball_t* a = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * K + 1));
    ball_t* b = (ball_t*)malloc(sizeof(ball_t) * (size_t)(K * N + 1));
    mat_load(a, A);
    mat_load(b, B);
    int W = block_width(a, M, K, b, N, lo, hi);
    int W2 = 2 * W + 1;
    uint64_t* ia = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M * (hi - lo) * W + 1));
    uint64_t* ib = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)((hi - lo) * N * W + 1));
    uint64_t* T = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M * N * W2 + 1));
    scale_block(a, M, K, b, N, lo, hi, row_scale, col_scale, W, ia, ib);
    int_gemm(ia, ib, M, hi - lo, N, W, T, W2);
    for (int64_t e = 0; e < M * N; e++) {
        const uint64_t* src = T + e * W2;
        uint64_t ext = (src[W2 - 1] >> 63) ? ~0ull : 0;
        for (int64_t q = 0; q < out_limbs; q++) out[e * out_limbs + q] = q < W2 ? src[q] : ext;
    }
    free(a);
    free(b);
    free(ia);
    free(ib);
    free(T);
    return g_status;
}

/* radius_matmul_upper (src/matmul.cpp:368-438) over Mag planes */
static void radius_mm(const mag_t* p, const mag_t* q, int64_t m, int64_t n, int64_t k, mag_t* c) {
    for (int64_t i = 0; i < m * k; i++) c[i] = mzero();
    int any_inf = 0;
    for (int64_t i = 0; i < m * n; i++) any_inf |= p[i].kind == MI;
    for (int64_t i = 0; i < n * k; i++) any_inf |= q[i].kind == MI;
    if (any_inf || n == 0) {
        for (int64_t i = 0; i < m; i++)
            for (int64_t j = 0; j < k; j++) {
                mag_t acc = mzero();
                for (int64_t l = 0; l < n; l++) acc = madd(acc, mmul(p[i * n + l], q[l * k + j]));
                c[i * k + j] = acc;
            }
        return;
    }
    win_t* ea = (win_t*)malloc(sizeof(win_t) * (size_t)(m * n + 1));
    win_t* eb = (win_t*)malloc(sizeof(win_t) * (size_t)(k * n + 1));
    for (int64_t i = 0; i < m; i++)
        for (int64_t l = 0; l < n; l++) {
            mag_t e = p[i * n + l];
            ea[i * n + l] = e.kind == MF ? (win_t){e.f, e.f - 30} : (win_t){INT64_MIN, INT64_MAX};
        }
    for (int64_t j = 0; j < k; j++)
        for (int64_t l = 0; l < n; l++) {
            mag_t e = q[l * k + j];
            eb[j * n + l] = e.kind == MF ? (win_t){e.f, e.f - 30} : (win_t){INT64_MIN, INT64_MAX};
        }
    int64_t* blocks = (int64_t*)malloc(sizeof(int64_t) * (size_t)(2 * n + 2));
    int64_t nb = greedy_split(n, m, k, ea, eb, 900, blocks);
    const mag_t infl = mparts((1ull << 29) + 1, 1);
    int64_t* ei = (int64_t*)malloc(sizeof(int64_t) * (size_t)(m + 1));
    int64_t* fj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(k + 1));
    for (int64_t bi = 0; bi < nb; bi++) {
        int64_t lo = blocks[2 * bi], hi = blocks[2 * bi + 1], w = hi - lo;
        for (int64_t i = 0; i < m; i++) {
            int64_t top = INT64_MIN, bot = INT64_MAX;
            for (int64_t l = lo; l < hi; l++) {
                win_t e = ea[i * n + l];
                if (e.top == INT64_MIN) continue;
                if (e.top > top) top = e.top;
                if (e.bot < bot) bot = e.bot;
            }
            ei[i] = top == INT64_MIN ? 0 : -((top + bot) / 2);
        }
        for (int64_t j = 0; j < k; j++) {
            int64_t top = INT64_MIN, bot = INT64_MAX;
            for (int64_t l = lo; l < hi; l++) {
                win_t e = eb[j * n + l];
                if (e.top == INT64_MIN) continue;
                if (e.top > top) top = e.top;
                if (e.bot < bot) bot = e.bot;
            }
            fj[j] = top == INT64_MIN ? 0 : -((top + bot) / 2);
        }
        double* da = (double*)malloc(sizeof(double) * (size_t)(m * w + 1));
        double* db = (double*)malloc(sizeof(double) * (size_t)(w * k + 1));
        for (int64_t i = 0; i < m; i++)
            for (int64_t l = 0; l < w; l++) da[i * w + l] = mldexp(p[i * n + lo + l], ei[i]);
        for (int64_t l = 0; l < w; l++)
            for (int64_t j = 0; j < k; j++) db[l * k + j] = mldexp(q[(lo + l) * k + j], fj[j]);
        for (int64_t i = 0; i < m; i++)
            for (int64_t j = 0; j < k; j++) {
                mag_t entry = mzero();
                for (int64_t c0 = 0; c0 < w; c0 += 1024) {
                    int64_t c1 = c0 + 1024 < w ? c0 + 1024 : w;
                    double s = 0.0;
                    for (int64_t l = c0; l < c1; l++) s += da[i * w + l] * db[l * k + j];
                    if (s != 0.0) entry = madd(entry, mmul(mfrom_double(s, -ei[i] - fj[j]), infl));
                }
                if (entry.kind != MZ) c[i * k + j] = madd(c[i * k + j], entry);
            }
        free(da);
        free(db);
    }
    free(ei);
    free(fj);
    free(blocks);
    free(ea);
    free(eb);
}

int orc_radius_matmul_upper(const uint32_t* pm, const int64_t* pe, const uint32_t* qm,
                            const int64_t* qe, int64_t m, int64_t n, int64_t k, uint32_t* om,
                            int64_t* oe) {
    g_status = APB_OK;
    mag_t* p = (mag_t*)malloc(sizeof(mag_t) * (size_t)(m * n + 1));
    mag_t* q = (mag_t*)malloc(sizeof(mag_t) * (size_t)(n * k + 1));
    mag_t* c = (mag_t*)malloc(sizeof(mag_t) * (size_t)(m * k + 1));
    for (int64_t i = 0; i < m * n; i++) p[i] = load_mag(pm[i], pe[i]);
    for (int64_t i = 0; i < n * k; i++) q[i] = load_mag(qm[i], qe[i]);
    radius_mm(p, q, m, n, k, c);
    for (int64_t i = 0; i < m * k; i++) {
        om[i] = c[i].kind == MZ ? 0 : (c[i].kind == MI ? APB_RAD_INF : (uint32_t)c[i].b);
        oe[i] = c[i].kind == MF ? c[i].f : 0;
    }
    free(p);
    free(q);
    free(c);
    return g_status;
}

/* classical_matmul_ball (src/matmul.cpp:442-451) */
static void classical(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N, int64_t p,
                      ball_t* c) {
    term_t* terms = (term_t*)malloc(sizeof(term_t) * (size_t)(K + 1));
    for (int64_t i = 0; i < M; i++)
        for (int64_t j = 0; j < N; j++) {
            for (int64_t k = 0; k < K; k++) terms[k] = (term_t){&a[i * K + k], &b[k * N + j], 0};
            dot_core(terms, K, p, 0, &c[i * N + j].m, &c[i * N + j].r, NULL, NULL, 0);
        }
    free(terms);
}

/* apfloat_from_bigint_scaled (src/bigint.cpp:187-191) of a two's complement value */
static void from_twos(of_t* out, const uint64_t* v, int W2, int64_t exp2) {
    uint64_t mag[2 * OL + 2];
    int neg = v[W2 - 1] >> 63;
    memcpy(mag, v, sizeof(uint64_t) * (size_t)W2);
    if (neg) {
        uint64_t c = 1;
        for (int q = 0; q < W2; q++) {
            uint64_t x = ~mag[q] + c;
            c = (c && x == 0);
            mag[q] = x;
        }
    }
    int nl = W2;
    while (nl > 0 && mag[nl - 1] == 0) nl--;
    if (nl == 0) {
        ozero(out);
        return;
    }
    onormalize(out, neg, 64 * (int64_t)nl + exp2, mag, nl);
}

/* block_matmul_ball (src/matmul.cpp:453-515) */
static void block_mm(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N, int64_t p,
                     ball_t* c, int64_t* nblocks) {
    for (int64_t i = 0; i < M * K; i++)
        if (!ofinite(&a[i].m) || a[i].r.kind == MI) {
            classical(a, M, K, b, N, p, c);
            return;
        }
    for (int64_t i = 0; i < K * N; i++)
        if (!ofinite(&b[i].m) || b[i].r.kind == MI) {
            classical(a, M, K, b, N, p, c);
            return;
        }
    int64_t* steps = (int64_t*)malloc(sizeof(int64_t) * (size_t)(3 * K + 3));
    int64_t ns = plan_blocks(a, M, K, b, N, p, steps);
    if (nblocks) *nblocks = ns;
    for (int64_t i = 0; i < M * N; i++) {
        ozero(&c[i].m);
        c[i].r = mzero();
    }
    term_t* terms = (term_t*)malloc(sizeof(term_t) * (size_t)(K + 2));
    static ball_t tmp, ex;
    for (int64_t s = 0; s < ns; s++) {
        int64_t lo = steps[3 * s], hi = steps[3 * s + 1], w = hi - lo;
        if (steps[3 * s + 2]) {
            for (int64_t i = 0; i < M; i++)
                for (int64_t j = 0; j < N; j++) {
                    for (int64_t k = 0; k < w; k++) terms[k] = (term_t){&a[i * K + lo + k], &b[(lo + k) * N + j], 0};
                    tmp = c[i * N + j];
                    terms[w] = (term_t){&tmp, &g_one, 0};
                    dot_core(terms, w + 1, p, 0, &c[i * N + j].m, &c[i * N + j].r, NULL, NULL, 0);
                }
            continue;
        }
        int W = block_width(a, M, K, b, N, lo, hi);
        int W2 = 2 * W + 1;
        int64_t* ei = (int64_t*)malloc(sizeof(int64_t) * (size_t)(M + 1));
        int64_t* fj = (int64_t*)malloc(sizeof(int64_t) * (size_t)(N + 1));
        uint64_t* ia = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M * w * W + 1));
        uint64_t* ib = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(w * N * W + 1));
        uint64_t* T = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(M * N * W2 + 1));
        scale_block(a, M, K, b, N, lo, hi, ei, fj, W, ia, ib);
        int_gemm(ia, ib, M, w, N, W, T, W2);
        for (int64_t i = 0; i < M; i++)
            for (int64_t j = 0; j < N; j++) {
                from_twos(&ex.m, T + (i * N + j) * W2, W2, -ei[i] - fj[j]);
                if (ex.m.kind == APB_ZERO) continue;
                ex.r = mzero();
                ball_add(&tmp, &c[i * N + j], &ex, p);
                c[i * N + j] = tmp;
            }
        free(ei);
        free(fj);
        free(ia);
        free(ib);
        free(T);
    }
    free(terms);
    free(steps);
    /* R_C += |A| R_B + R_A (|B| + R_B) (src/matmul.cpp:498-513) */
    mag_t* abs_a = (mag_t*)malloc(sizeof(mag_t) * (size_t)(M * K + 1));
    mag_t* rad_a = (mag_t*)malloc(sizeof(mag_t) * (size_t)(M * K + 1));
    mag_t* rad_b = (mag_t*)malloc(sizeof(mag_t) * (size_t)(K * N + 1));
    mag_t* absrad_b = (mag_t*)malloc(sizeof(mag_t) * (size_t)(K * N + 1));
    mag_t* r1 = (mag_t*)malloc(sizeof(mag_t) * (size_t)(M * N + 1));
    mag_t* r2 = (mag_t*)malloc(sizeof(mag_t) * (size_t)(M * N + 1));
    for (int64_t i = 0; i < M * K; i++) {
        abs_a[i] = a[i].m.kind == APB_ZERO ? mzero() : mupper(&a[i].m);
        rad_a[i] = a[i].r;
    }
    for (int64_t i = 0; i < K * N; i++) {
        rad_b[i] = b[i].r;
        absrad_b[i] = madd(b[i].m.kind == APB_ZERO ? mzero() : mupper(&b[i].m), b[i].r);
    }
    radius_mm(abs_a, rad_b, M, K, N, r1);
    radius_mm(rad_a, absrad_b, M, K, N, r2);
    for (int64_t i = 0; i < M * N; i++) c[i].r = madd(c[i].r, madd(r1[i], r2[i]));
    free(abs_a);
    free(rad_a);
    free(rad_b);
    free(absrad_b);
    free(r1);
    free(r2);
}

/* matmul_dispatch_cutoff (src/matmul.cpp:517-524) */
static int64_t cutoff(int64_t p) {
    if (p <= 64) return 60;
    if (p <= 128) return 56;
    if (p <= 256) return 52;
    if (p <= 512) return 48;
    if (p <= 1024) return 44;
    return 40;
}

static void matmul_any(const ball_t* a, int64_t M, int64_t K, const ball_t* b, int64_t N, int64_t p,
                       int algo, ball_t* c, int64_t* nblocks) {
    if (nblocks) *nblocks = 0;
    if (algo == APB_MM_CLASSICAL) {
        classical(a, M, K, b, N, p, c);
        return;
    }
    if (algo == APB_MM_AUTO) {
        int64_t mind = M < K ? M : K;
        if (N < mind) mind = N;
        if (mind <= cutoff(p)) {
            classical(a, M, K, b, N, p, c);
            return;
        }
    }
    block_mm(a, M, K, b, N, p, c, nblocks);
}

int orc_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
               int64_t* block_count) {
    g_status = APB_OK;
    if (A->cols != B->rows) return APB_ERR_INVALID;
    init_one();
    const int64_t M = A->rows, K = A->cols, N = B->cols;
    ball_t* a = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * K + 1));
    ball_t* b = (ball_t*)malloc(sizeof(ball_t) * (size_t)(K * N + 1));
    ball_t* c = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * N + 1));
    mat_load(a, A);
    mat_load(b, B);
    matmul_any(a, M, K, b, N, prec, algo, c, block_count);
    for (int64_t i = 0; i < M * N; i++) store_ball(&C->b, i, &c[i].m, c[i].r);
    free(a);
    free(b);
    free(c);
    return g_status;
}

/* complex_matmul_ball (src/matmul.cpp:533-548) */
int orc_matmul_complex(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                       const apb_mat* Bim, int64_t prec, apb_mat* Cre, apb_mat* Cim) {
    g_status = APB_OK;
    if (Are->cols != Bre->rows) return APB_ERR_INVALID;
    init_one();
    const int64_t M = Are->rows, K = Are->cols, N = Bre->cols;
    ball_t* ar = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * K + 1));
    ball_t* ai = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * K + 1));
    ball_t* br = (ball_t*)malloc(sizeof(ball_t) * (size_t)(K * N + 1));
    ball_t* bi = (ball_t*)malloc(sizeof(ball_t) * (size_t)(K * N + 1));
    ball_t* p4[4];
    for (int q = 0; q < 4; q++) p4[q] = (ball_t*)malloc(sizeof(ball_t) * (size_t)(M * N + 1));
    mat_load(ar, Are);
    mat_load(ai, Aim);
    mat_load(br, Bre);
    mat_load(bi, Bim);
    matmul_any(ar, M, K, br, N, prec, APB_MM_AUTO, p4[0], NULL); /* AC */
    matmul_any(ai, M, K, bi, N, prec, APB_MM_AUTO, p4[1], NULL); /* BD */
    matmul_any(ar, M, K, bi, N, prec, APB_MM_AUTO, p4[2], NULL); /* AD */
    matmul_any(ai, M, K, br, N, prec, APB_MM_AUTO, p4[3], NULL); /* BC */
    static ball_t r, nb;
    for (int64_t i = 0; i < M * N; i++) {
        nb = p4[1][i];
        oneg(&nb.m);
        ball_add(&r, &p4[0][i], &nb, prec);
        store_ball(&Cre->b, i, &r.m, r.r);
        ball_add(&r, &p4[2][i], &p4[3][i], prec);
        store_ball(&Cim->b, i, &r.m, r.r);
    }
    free(ar);
    free(ai);
    free(br);
    free(bi);
    for (int q = 0; q < 4; q++) free(p4[q]);
    return g_status;
}

/* ------------------------------------------------------------ poly */
/* poly_mullow_classical (src/poly.cpp:11-26): coefficient k is one fused dot
 * over (a_i, b_{k-i}), i in [max(0, k+1-|b|), min(k, |a|-1)] */
int orc_poly_mullow(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                    int64_t prec, apb_balls* out) {
    g_status = APB_OK;
    init_one();
    int64_t nmax = alen < blen ? alen : blen;
    if (nmax < 1) nmax = 1;
    ball_t* xs = (ball_t*)malloc(sizeof(ball_t) * (size_t)nmax);
    ball_t* ys = (ball_t*)malloc(sizeof(ball_t) * (size_t)nmax);
    term_t* terms = (term_t*)malloc(sizeof(term_t) * (size_t)nmax);
    static of_t mid;
    for (int64_t k = 0; k < len; k++) {
        of_t z;
        ozero(&z);
        if (alen == 0 || blen == 0) {
            store_ball(out, k, &z, mzero());
            continue;
        }
        const int64_t i0 = k + 1 > blen ? k + 1 - blen : 0;
        const int64_t i1 = k < alen - 1 ? k : alen - 1;
        if (i0 >= alen || i1 < i0) {
            store_ball(out, k, &z, mzero());
            continue;
        }
        const int64_t n = i1 - i0 + 1;
        for (int64_t i = 0; i < n; i++) {
            load_ball(&xs[i], a, i0 + i);
            load_ball(&ys[i], b, k - i0 - i);
            terms[i].x = &xs[i];
            terms[i].y = &ys[i];
            terms[i].neg = 0;
        }
        mag_t rad;
        dot_core(terms, n, prec, 0, &mid, &rad, NULL, NULL, 0);
        store_ball(out, k, &mid, rad);
    }
    free(xs);
    free(ys);
    free(terms);
    return g_status;
}

/* apfloat_mul_u64_exact (src/apfloat.cpp:178-186) */
static void omul_u64_exact(of_t* out, const of_t* x, uint64_t k) {
    if (x->kind != APB_FINITE) {
        *out = *x;
        if (k == 0 && (x->kind == APB_PINF || x->kind == APB_NINF)) out->kind = APB_NAN;
        return;
    }
    if (k == 0) {
        ozero(out);
        return;
    }
    uint64_t prod[OL];
    uint64_t cy = 0;
    for (int i = 0; i < x->n; i++) {
        const u128 t = (u128)x->d[i] * k + cy;
        prod[i] = (uint64_t)t;
        cy = (uint64_t)(t >> 64);
    }
    prod[x->n] = cy;
    onormalize(out, x->neg, checked_exp((i128)x->e + 64), prod, x->n + 1);
}

/* mag_inv_u64_upper (src/mag.cpp:155-164) */
static mag_t minv_u64(uint64_t k) {
    const unsigned len = bitw(k);
    if ((k & (k - 1)) == 0) return mparts(MAG_ONE >> 1, 2 - (int64_t)len);
    const u128 num = (u128)1 << (30 - 1 + len);
    uint64_t q = (uint64_t)(num / k);
    if (num % k) q++;
    return mparts(q, 1 - (int64_t)len);
}

/* ball_div_u64 (src/ball.cpp:38-43) over apfloat_div_u64 (src/apfloat.cpp:308-331) */
static void ball_div_u64(ball_t* r, const ball_t* x, uint64_t k, int64_t p) {
    if (x->m.kind == APB_NAN) {
        set_indeterminate(r);
        return;
    }
    if (p < 2) p = 2;
    mag_t err = mzero();
    if (x->m.kind != APB_FINITE) {
        r->m = x->m;
    } else {
        const int n = x->m.n;
        const int64_t wl = (int64_t)n > p / 64 + 1 ? (int64_t)n : p / 64 + 1;
        const int w = (int)wl + 1;
        uint64_t q[OL] = {0};
        uint64_t rem = 0;
        for (int i = w - 1; i >= 0; i--) {
            const uint64_t num = i + n >= w ? x->m.d[i + n - w] : 0;
            const u128 cur = ((u128)rem << 64) | num;
            q[i] = (uint64_t)(cur / k);
            rem = (uint64_t)(cur % k);
        }
        onormalize(&r->m, x->m.neg, x->m.e, q, w);
        err = oround(&r->m, p);
        if (rem) err = madd(err, mfrom_u64(1, checked_exp((i128)x->m.e - 64 * (i128)w)));
    }
    r->r = madd(err, mmul(x->r, minv_u64(k)));
}

/* series_exp_basecase (src/poly.cpp:28-46); APB_ERR_INVALID for the reference's
 * std::domain_error on a constant term that is not an exact zero */
int orc_series_exp(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out) {
    g_status = APB_OK;
    init_one();
    if (alen > 0 && ((a->kind[0] & APB_KIND_MASK) != APB_ZERO || a->rad_man[0] != 0)) return APB_ERR_INVALID;
    if (len == 0) return APB_OK;
    ball_t* b = (ball_t*)malloc(sizeof(ball_t) * (size_t)len);
    ball_t* ja = (ball_t*)malloc(sizeof(ball_t) * (size_t)len);
    term_t* terms = (term_t*)malloc(sizeof(term_t) * (size_t)len);
    for (int64_t j = 0; j < len; j++) {
        ozero(&ja[j].m);
        ja[j].r = mzero();
        if (j >= 1 && j < alen) {
            static ball_t aj;
            load_ball(&aj, a, j);
            omul_u64_exact(&ja[j].m, &aj.m, (uint64_t)j);
            ja[j].r = mmul(aj.r, mfrom_u64((uint64_t)j, 0));
        }
    }
    b[0] = g_one;
    for (int64_t k = 1; k < len; k++) {
        for (int64_t i = 0; i < k; i++) {
            terms[i].x = &ja[1 + i];
            terms[i].y = &b[k - 1 - i];
            terms[i].neg = 0;
        }
        static ball_t s;
        dot_core(terms, k, prec, 0, &s.m, &s.r, NULL, NULL, 0);
        ball_div_u64(&b[k], &s, (uint64_t)k, prec);
    }
    for (int64_t k = 0; k < len; k++) store_ball(out, k, &b[k].m, b[k].r);
    free(b);
    free(ja);
    free(terms);
    return g_status;
}

