// apball_b200.hpp - header-only C++ drop-in for the reference `apball` API
// (/root/reference/proj/include/apball/{dot,matmul}.hpp) on top of the C ABI
// of libapb_b200.so (include/apb.h).
//
// A caller of the reference switches by including this header next to the
// reference headers and calling apball::b200::<op> with the reference's own
// types and argument meaning; the bodies pack the AoS balls into the SoA
// layout of apb.h, run the B200 kernels (host->device copies inside), unpack,
// and map status codes back to the reference's exceptions:
//   APB_ERR_INVALID -> std::invalid_argument, APB_ERR_OVERFLOW -> std::overflow_error.
//
// Replaced interfaces (reference file:line):
//   dot_ball            include/apball/dot.hpp:73-74   (src/dot.cpp:402-405)
//   dot_approx          include/apball/dot.hpp:77-78
//   dot_complex_ball / dot_complex_approx  include/apball/dot.hpp:86-89
//   block_matmul_ball   include/apball/matmul.hpp:90   (src/matmul.cpp:453-515)
//   matmul_auto         include/apball/matmul.hpp:91
//   classical_matmul_ball include/apball/matmul.hpp:89
//   complex_matmul_ball include/apball/matmul.hpp:92-93
//   poly_mullow_classical include/apball/poly.hpp:23-24  (src/poly.cpp:11-26)
//   series_exp_basecase include/apball/poly.hpp:27-29    (src/poly.cpp:28-46)
#pragma once

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "apb.h"
#include "apball/ball.hpp"
#include "apball/dot.hpp"
#include "apball/matmul.hpp"
#include "apball/poly.hpp"

namespace apball::b200 {

namespace detail {

struct SoA {
    std::vector<uint64_t> mant;
    std::vector<int64_t> exp, rad_exp;
    std::vector<uint8_t> kind;
    std::vector<uint32_t> rad_man;
    int32_t L = 1;
    apb_balls view() {
        return apb_balls{mant.data(), exp.data(), kind.data(), rad_man.data(), rad_exp.data(),
                         (int64_t)exp.size(), L};
    }
    void resize(size_t n, int32_t l) {
        L = l < 1 ? 1 : l;
        mant.assign(n * (size_t)L, 0);
        exp.assign(n, 0);
        rad_exp.assign(n, 0);
        kind.assign(n, 0);
        rad_man.assign(n, 0);
    }
};

inline int32_t limbs_needed(const Ball* const* balls, size_t n) {
    size_t L = 1;
    for (size_t i = 0; i < n; i++)
        if (balls[i]->mid.is_finite() && !balls[i]->mid.is_zero()) L = std::max(L, balls[i]->mid.limb_count());
    return (int32_t)L;
}

inline void put(SoA& s, size_t e, const Ball& b) {
    const ApFloat& m = b.mid;
    switch (m.kind()) {
        case FloatKind::Zero: s.kind[e] = APB_ZERO; break;
        case FloatKind::PosInf: s.kind[e] = APB_PINF; break;
        case FloatKind::NegInf: s.kind[e] = APB_NINF; break;
        case FloatKind::NaN: s.kind[e] = APB_NAN; break;
        default: {
            const size_t n = m.limb_count();
            for (size_t i = 0; i < n; i++) s.mant[e * (size_t)s.L + (size_t)s.L - n + i] = m.limbs()[i];
            s.exp[e] = m.exponent();
            s.kind[e] = (uint8_t)(APB_FINITE | (m.negative() ? APB_SIGN : 0));
        }
    }
    if (b.rad.is_zero()) {
        s.rad_man[e] = 0;
    } else if (b.rad.is_inf()) {
        s.rad_man[e] = APB_RAD_INF;
    } else {
        s.rad_man[e] = (uint32_t)b.rad.mantissa();
        s.rad_exp[e] = b.rad.exponent();
    }
}

inline Ball get(const SoA& s, size_t e) {
    Ball b;
    switch (s.kind[e] & APB_KIND_MASK) {
        case APB_ZERO: break;
        case APB_PINF: b.mid = ApFloat::pos_inf(); break;
        case APB_NINF: b.mid = ApFloat::neg_inf(); break;
        case APB_NAN: b.mid = ApFloat::nan(); break;
        default: {
            const uint64_t* m = s.mant.data() + e * (size_t)s.L;
            size_t z = 0;
            while (z < (size_t)s.L && m[z] == 0) z++;
            LimbVec v;
            v.assign(m + z, (size_t)s.L - z);
            b.mid = ApFloat::from_normalized((s.kind[e] & APB_SIGN) != 0, s.exp[e], std::move(v));
        }
    }
    const uint32_t rb = s.rad_man[e];
    b.rad = rb == 0 ? Mag::zero() : (rb == APB_RAD_INF ? Mag::inf() : Mag::from_parts(rb, s.rad_exp[e]));
    return b;
}

inline void check(int rc, bool domain = false) {
    if (rc == APB_OK) return;
    std::string msg = apb_last_error();
    if (domain && rc == APB_ERR_INVALID) throw std::domain_error(msg);
    if (rc == APB_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == APB_ERR_OVERFLOW) throw std::overflow_error(msg);
    throw std::runtime_error("apb: " + msg);
}

inline void pack_matrix(SoA& s, const BallMatrix& m) {
    std::vector<const Ball*> ptr(m.a.size());
    for (size_t i = 0; i < m.a.size(); i++) ptr[i] = &m.a[i];
    s.resize(m.a.size(), limbs_needed(ptr.data(), ptr.size()));
    for (size_t i = 0; i < m.a.size(); i++) put(s, i, m.a[i]);
}

inline BallMatrix unpack_matrix(const SoA& s, size_t rows, size_t cols) {
    BallMatrix m(rows, cols);
    for (size_t i = 0; i < rows * cols; i++) m.a[i] = get(s, i);
    return m;
}

inline Ball dot_impl(const Ball* initial, bool subtract, const Ball* x, std::ptrdiff_t xstep,
                     const Ball* y, std::ptrdiff_t ystep, std::size_t n, std::int64_t p, int mode) {
    std::vector<const Ball*> px(n), py(n);
    for (size_t i = 0; i < n; i++) {
        px[i] = x + (std::ptrdiff_t)i * xstep;
        py[i] = y + (std::ptrdiff_t)i * ystep;
    }
    SoA sx, sy, si, so;
    sx.resize(n ? n : 1, limbs_needed(px.data(), n));
    sy.resize(n ? n : 1, limbs_needed(py.data(), n));
    for (size_t i = 0; i < n; i++) {
        put(sx, i, *px[i]);
        put(sy, i, *py[i]);
    }
    if (initial) {
        const Ball* pi = initial;
        si.resize(1, limbs_needed(&pi, 1));
        put(si, 0, *initial);
    }
    so.resize(1, (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64));
    apb_balls vx = sx.view(), vy = sy.view(), vi = si.view(), vo = so.view();
    apb_dot_index idx{1, 0, (int64_t)n, 0, 1, 0, (int64_t)n, 0, 1};
    check(apb_dot_batch_host(&vx, &vy, initial ? &vi : nullptr, subtract ? 1 : 0, &idx, (int64_t)n, 1, p,
                             mode, &vo));
    return get(so, 0);
}

}  // namespace detail

inline Ball dot_ball(const Ball* initial, bool subtract, const Ball* x, std::ptrdiff_t xstep,
                     const Ball* y, std::ptrdiff_t ystep, std::size_t n, std::int64_t p) {
    return detail::dot_impl(initial, subtract, x, xstep, y, ystep, n, p, APB_DOT_BALL);
}

inline ApFloat dot_approx(const Ball* initial, bool subtract, const Ball* x, std::ptrdiff_t xstep,
                          const Ball* y, std::ptrdiff_t ystep, std::size_t n, std::int64_t p) {
    return detail::dot_impl(initial, subtract, x, xstep, y, ystep, n, p, APB_DOT_APPROX).mid;
}

// dot_complex_ball / dot_complex_approx (dot.hpp:86-89): the reference's
// dot_tuning() knobs are honoured and dot_threeprod_hits() is advanced by the
// number of terms passing the three-multiplication gate (src/dot.cpp:494-501)
inline ComplexBall complex_dot_impl(const ComplexBall* x, std::ptrdiff_t xstep, const ComplexBall* y,
                                    std::ptrdiff_t ystep, std::size_t n, std::int64_t p, int mode) {
    std::vector<const Ball*> pxr(n), pxi(n), pyr(n), pyi(n);
    for (size_t i = 0; i < n; i++) {
        pxr[i] = &x[(std::ptrdiff_t)i * xstep].re;
        pxi[i] = &x[(std::ptrdiff_t)i * xstep].im;
        pyr[i] = &y[(std::ptrdiff_t)i * ystep].re;
        pyi[i] = &y[(std::ptrdiff_t)i * ystep].im;
    }
    const std::vector<const Ball*>* pp[4] = {&pxr, &pxi, &pyr, &pyi};
    detail::SoA s[4], ore, oim;
    for (int q = 0; q < 4; q++) {
        s[q].resize(n ? n : 1, detail::limbs_needed(pp[q]->data(), n));
        for (size_t i = 0; i < n; i++) detail::put(s[q], i, *(*pp[q])[i]);
    }
    const int32_t L = (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64);
    ore.resize(1, L);
    oim.resize(1, L);
    apb_balls v[4] = {s[0].view(), s[1].view(), s[2].view(), s[3].view()};
    apb_balls vr = ore.view(), vi = oim.view();
    apb_dot_index idx{1, 0, (int64_t)n, 0, 1, 0, (int64_t)n, 0, 1};
    const DotTuning& t = dot_tuning();
    apb_dot_tuning tun{t.disable_precision_reduction ? 1 : 0, t.force_threeprod ? 1 : 0,
                       (int64_t)std::min<std::size_t>(t.threeprod_cutoff_limbs, (std::size_t)INT64_MAX)};
    uint64_t hits = 0;
    detail::check(apb_dot_complex_batch_host(&v[0], &v[1], &v[2], &v[3], &idx, (int64_t)n, 1, p, mode, &tun, &vr,
                                             &vi, &hits));
    dot_threeprod_hits() += hits;
    return ComplexBall{detail::get(ore, 0), detail::get(oim, 0)};
}

inline ComplexBall dot_complex_ball(const ComplexBall* x, std::ptrdiff_t xstep, const ComplexBall* y,
                                    std::ptrdiff_t ystep, std::size_t n, std::int64_t p) {
    return complex_dot_impl(x, xstep, y, ystep, n, p, APB_DOT_BALL);
}

inline ApComplex dot_complex_approx(const ComplexBall* x, std::ptrdiff_t xstep, const ComplexBall* y,
                                    std::ptrdiff_t ystep, std::size_t n, std::int64_t p) {
    ComplexBall r = complex_dot_impl(x, xstep, y, ystep, n, p, APB_DOT_APPROX);
    return ApComplex{r.re.mid, r.im.mid};
}

inline BallMatrix matmul_with(const BallMatrix& a, const BallMatrix& b, std::int64_t p, int algo) {
    if (a.cols != b.rows) throw std::invalid_argument("matmul: dimension mismatch");
    detail::SoA sa, sb, sc;
    detail::pack_matrix(sa, a);
    detail::pack_matrix(sb, b);
    sc.resize(a.rows * b.cols, (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64));
    apb_mat A{sa.view(), (int64_t)a.rows, (int64_t)a.cols}, B{sb.view(), (int64_t)b.rows, (int64_t)b.cols};
    apb_mat C{sc.view(), (int64_t)a.rows, (int64_t)b.cols};
    detail::check(apb_matmul_host(&A, &B, p, algo, &C));
    return detail::unpack_matrix(sc, a.rows, b.cols);
}

inline BallMatrix block_matmul_ball(const BallMatrix& a, const BallMatrix& b, std::int64_t p) {
    return matmul_with(a, b, p, APB_MM_BLOCK);
}
inline BallMatrix classical_matmul_ball(const BallMatrix& a, const BallMatrix& b, std::int64_t p) {
    return matmul_with(a, b, p, APB_MM_CLASSICAL);
}
inline BallMatrix matmul_auto(const BallMatrix& a, const BallMatrix& b, std::int64_t p) {
    return matmul_with(a, b, p, APB_MM_AUTO);
}

// complex_matmul_ball: four real products + re/im combine, all on the device
// (src/matmul.cpp:533-548)
inline ComplexBallMatrix complex_matmul_ball(const ComplexBallMatrix& a, const ComplexBallMatrix& b,
                                             std::int64_t p) {
    if (a.cols != b.rows) throw std::invalid_argument("matmul: dimension mismatch");
    detail::SoA s[6];
    detail::pack_matrix(s[0], a.real_part());
    detail::pack_matrix(s[1], a.imag_part());
    detail::pack_matrix(s[2], b.real_part());
    detail::pack_matrix(s[3], b.imag_part());
    const int32_t L = (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64);
    s[4].resize(a.rows * b.cols, L);
    s[5].resize(a.rows * b.cols, L);
    apb_mat m[6] = {{s[0].view(), (int64_t)a.rows, (int64_t)a.cols}, {s[1].view(), (int64_t)a.rows, (int64_t)a.cols},
                    {s[2].view(), (int64_t)b.rows, (int64_t)b.cols}, {s[3].view(), (int64_t)b.rows, (int64_t)b.cols},
                    {s[4].view(), (int64_t)a.rows, (int64_t)b.cols}, {s[5].view(), (int64_t)a.rows, (int64_t)b.cols}};
    detail::check(apb_matmul_complex_host(&m[0], &m[1], &m[2], &m[3], p, APB_MM_AUTO, &m[4], &m[5]));
    return ComplexBallMatrix::from_parts(detail::unpack_matrix(s[4], a.rows, b.cols),
                                         detail::unpack_matrix(s[5], a.rows, b.cols));
}

// poly_mullow_classical: one batched launch of variable-length negative-stride dots
inline BallPoly poly_mullow_classical(const BallPoly& a, const BallPoly& b, std::size_t len, std::int64_t p) {
    detail::SoA sa, sb, so;
    std::vector<const Ball*> pa(a.c.size()), pb(b.c.size());
    for (size_t i = 0; i < a.c.size(); i++) pa[i] = &a.c[i];
    for (size_t i = 0; i < b.c.size(); i++) pb[i] = &b.c[i];
    sa.resize(a.c.size() ? a.c.size() : 1, detail::limbs_needed(pa.data(), pa.size()));
    sb.resize(b.c.size() ? b.c.size() : 1, detail::limbs_needed(pb.data(), pb.size()));
    for (size_t i = 0; i < a.c.size(); i++) detail::put(sa, i, a.c[i]);
    for (size_t i = 0; i < b.c.size(); i++) detail::put(sb, i, b.c[i]);
    so.resize(len ? len : 1, (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64));
    apb_balls va = sa.view(), vb = sb.view(), vo = so.view();
    detail::check(apb_poly_mullow_host(&va, (int64_t)a.c.size(), &vb, (int64_t)b.c.size(), (int64_t)len, p, &vo));
    BallPoly out = BallPoly::zero(len);
    for (size_t k = 0; k < len; k++) out.c[k] = detail::get(so, k);
    return out;
}

// series_exp_basecase: std::domain_error unless a.c[0] is an exact zero
inline BallPoly series_exp_basecase(const BallPoly& a, std::size_t len, std::int64_t p) {
    detail::SoA sa, so;
    std::vector<const Ball*> pa(a.c.size());
    for (size_t i = 0; i < a.c.size(); i++) pa[i] = &a.c[i];
    sa.resize(a.c.size() ? a.c.size() : 1, detail::limbs_needed(pa.data(), pa.size()));
    for (size_t i = 0; i < a.c.size(); i++) detail::put(sa, i, a.c[i]);
    so.resize(len ? len : 1, (int32_t)((std::max<std::int64_t>(p, 2) + 63) / 64));
    apb_balls va = sa.view(), vo = so.view();
    detail::check(apb_series_exp_host(&va, (int64_t)a.c.size(), (int64_t)len, p, &vo), true);
    BallPoly out = BallPoly::zero(len);
    for (size_t k = 0; k < len; k++) out.c[k] = detail::get(so, k);
    return out;
}

}  // namespace apball::b200
