// ref_shim.cpp - TEST INFRASTRUCTURE ONLY (oracle side; never shipped, never on
// the product path).
//
// A flat extern "C" surface over the UNMODIFIED reference library `apball`
// (compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref),
// speaking the SoA ball layout of include/apb.h.  Used to
//   * generate the golden fixtures under tests/golden (oracle/gen_golden.py),
//   * check the GPU results against the reference itself on the GPU box
//     (oracle/_ref travels with the snapshot; /root/reference does not),
//   * time the reference CPU path for bench.py's cpu_baseline / --impl reference.
// Every function calls the reference's own public API; nothing here
// re-implements its arithmetic except the conversion between layouts.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "apball/ball.hpp"
#include "apball/bench.hpp"
#include "apball/dot.hpp"
#include "apball/matmul.hpp"
#include "apball/oracle.hpp"
#include "apball/poly.hpp"
#include "apb.h"

using namespace apball;

namespace {

thread_local std::string g_err;

ApFloat load_mid(const apb_balls* a, int64_t e) {
    const uint8_t k = a->kind[e];
    switch (k & APB_KIND_MASK) {
        case APB_ZERO: return ApFloat::zero();
        case APB_PINF: return ApFloat::pos_inf();
        case APB_NINF: return ApFloat::neg_inf();
        case APB_NAN: return ApFloat::nan();
        default: break;
    }
    const uint64_t* m = a->mant + e * int64_t(a->L);
    int z = 0;
    while (z < a->L && m[z] == 0) z++;
    LimbVec v;
    v.assign(m + z, size_t(a->L - z));
    return ApFloat::from_normalized((k & APB_SIGN) != 0, a->exp[e], std::move(v));
}

Mag load_rad(const apb_balls* a, int64_t e) {
    uint32_t b = a->rad_man[e];
    if (b == 0) return Mag::zero();
    if (b == APB_RAD_INF) return Mag::inf();
    return Mag::from_parts(b, a->rad_exp[e]);
}

Ball load_ball(const apb_balls* a, int64_t e) { return Ball{load_mid(a, e), load_rad(a, e)}; }

void store_mid(apb_balls* a, int64_t e, const ApFloat& x) {
    uint64_t* m = a->mant + e * int64_t(a->L);
    std::memset(m, 0, sizeof(uint64_t) * size_t(a->L));
    a->exp[e] = 0;
    switch (x.kind()) {
        case FloatKind::Zero: a->kind[e] = APB_ZERO; return;
        case FloatKind::PosInf: a->kind[e] = APB_PINF; return;
        case FloatKind::NegInf: a->kind[e] = APB_NINF; return;
        case FloatKind::NaN: a->kind[e] = APB_NAN; return;
        default: break;
    }
    const size_t n = x.limb_count();
    if (int64_t(n) > a->L) throw std::length_error("ref_shim: output limb slot too small");
    for (size_t i = 0; i < n; i++) m[size_t(a->L) - n + i] = x.limbs()[i];
    a->exp[e] = x.exponent();
    a->kind[e] = uint8_t(APB_FINITE | (x.negative() ? APB_SIGN : 0));
}

void store_rad(apb_balls* a, int64_t e, const Mag& r) {
    if (r.is_zero()) {
        a->rad_man[e] = 0;
        a->rad_exp[e] = 0;
    } else if (r.is_inf()) {
        a->rad_man[e] = APB_RAD_INF;
        a->rad_exp[e] = 0;
    } else {
        a->rad_man[e] = uint32_t(r.mantissa());
        a->rad_exp[e] = r.exponent();
    }
}

void store_ball(apb_balls* a, int64_t e, const Ball& b) {
    store_mid(a, e, b.mid);
    store_rad(a, e, b.rad);
}

int64_t x_elem(const apb_dot_index* ix, int64_t b, int64_t i) {
    return ix->x_off + (b / ix->bdiv) * ix->xs1 + (b % ix->bdiv) * ix->xs2 + i * ix->xstep;
}
int64_t y_elem(const apb_dot_index* ix, int64_t b, int64_t i) {
    return ix->y_off + (b / ix->bdiv) * ix->ys1 + (b % ix->bdiv) * ix->ys2 + i * ix->ystep;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return APB_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return APB_ERR_INVALID;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return APB_ERR_OVERFLOW;
    } catch (const std::domain_error& e) {  // series_exp_basecase's constant-term check
        g_err = e.what();
        return APB_ERR_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return APB_ERR_UNSUPPORTED;
    }
}

template <class F>
void parallel_for(int64_t n, int threads, F&& f) {
    if (threads <= 1 || n < 2) {
        f(int64_t(0), n);
        return;
    }
    threads = int(std::min<int64_t>(threads, n));
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(static_cast<size_t>(threads));
    std::exception_ptr* ep = errs.data();
    for (int t = 0; t < threads; t++) {
        int64_t lo = n * t / threads, hi = n * (t + 1) / threads;
        pool.emplace_back([&f, ep, lo, hi, t]() {
            try {
                f(lo, hi);
            } catch (...) {
                ep[t] = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
}

BallMatrix load_matrix(const apb_mat* m) {
    BallMatrix r(static_cast<size_t>(m->rows), static_cast<size_t>(m->cols));
    for (int64_t i = 0; i < m->rows * m->cols; i++) r.a[size_t(i)] = load_ball(&m->b, i);
    return r;
}

void store_matrix(apb_mat* m, const BallMatrix& r) {
    for (int64_t i = 0; i < m->rows * m->cols; i++) store_ball(&m->b, i, r.a[size_t(i)]);
}

MagMatrix load_mags(const uint32_t* man, const int64_t* ex, int64_t r, int64_t c) {
    MagMatrix m(static_cast<size_t>(r), static_cast<size_t>(c));
    for (int64_t i = 0; i < r * c; i++) {
        uint32_t b = man[i];
        m.a[size_t(i)] = b == 0 ? Mag::zero() : (b == APB_RAD_INF ? Mag::inf() : Mag::from_parts(b, ex[i]));
    }
    return m;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// dot_ball / dot_approx per dot (src/dot.cpp:402-410), batch split over threads
int ref_dot_batch(const apb_balls* x, const apb_balls* y, const apb_balls* initial, int subtract,
                  const apb_dot_index* ix, int64_t n, int64_t batch, int64_t prec, int mode,
                  int disable_reduction, apb_balls* out, int threads) {
    return guarded([&] {
        parallel_for(batch, threads, [&](int64_t lo, int64_t hi) {
            dot_tuning().disable_precision_reduction = disable_reduction != 0;
            std::vector<Ball> xs(static_cast<size_t>(n)), ys(static_cast<size_t>(n));
            for (int64_t b = lo; b < hi; b++) {
                for (int64_t i = 0; i < n; i++) {
                    xs[size_t(i)] = load_ball(x, x_elem(ix, b, i));
                    ys[size_t(i)] = load_ball(y, y_elem(ix, b, i));
                }
                Ball init;
                if (initial) init = load_ball(initial, b);
                if (mode == APB_DOT_APPROX) {
                    ApFloat r = dot_approx(initial ? &init : nullptr, subtract != 0, xs.data(), 1,
                                           ys.data(), 1, size_t(n), prec);
                    store_ball(out, b, Ball::exact(r));
                } else {
                    Ball r = dot_ball(initial ? &init : nullptr, subtract != 0, xs.data(), 1,
                                      ys.data(), 1, size_t(n), prec);
                    store_ball(out, b, r);
                }
            }
            dot_tuning().disable_precision_reduction = false;
        });
    });
}

// dot_setup -> dot_init -> dot_accumulate_term / dot_accumulate_radius
// (include/apball/dot.hpp:57-67): plan + accumulator state BEFORE finalize.
int ref_dot_state(const apb_balls* x, const apb_balls* y, const apb_balls* initial, int subtract,
                  const apb_dot_index* ix, int64_t n, int64_t batch, int64_t prec,
                  int disable_reduction, apb_dot_state* st, uint64_t* acc, int64_t acc_stride) {
    return guarded([&] {
        dot_tuning().disable_precision_reduction = disable_reduction != 0;
        std::vector<std::pair<Ball, Ball>> terms;
        for (int64_t b = 0; b < batch; b++) {
            terms.clear();
            for (int64_t i = 0; i < n; i++)
                terms.emplace_back(load_ball(x, x_elem(ix, b, i)), load_ball(y, y_elem(ix, b, i)));
            if (initial) terms.emplace_back(load_ball(initial, b), Ball::from_i64(1));
            DotPlan plan = dot_setup(terms, prec);
            apb_dot_state& s = st[b];
            std::memset(&s, 0, sizeof s);
            s.e_max = plan.e_max;
            s.e_min = plan.e_min;
            s.e_rad = plan.e_rad;
            s.n_nonzero = plan.n_nonzero;
            s.p_eff = plan.p_eff;
            s.extend = int32_t(plan.extend);
            s.padding = int32_t(plan.padding);
            s.n_s = int64_t(plan.n_s);
            s.e_s = plan.e_s;
            s.status = int32_t(plan.status);
            if (plan.status != DotStatus::Proceed) continue;
            DotAccumulator a;
            dot_init(plan, a);
            for (size_t i = 0; i < terms.size(); i++) {
                const Ball& u = terms[i].first;
                const Ball& v = terms[i].second;
                bool neg = (int64_t(i) < n) && subtract;
                if (!u.mid.is_zero() && !v.mid.is_zero())
                    dot_accumulate_term(plan, a, u.mid, v.mid, neg);
                // radius terms |m|r', |m'|r, r r' (src/dot.cpp:346-358)
                if (!v.rad.is_zero() && !u.mid.is_zero())
                    dot_accumulate_radius(a, mag_upper_from_apfloat(u.mid), v.rad, plan.e_rad);
                if (!u.rad.is_zero() && !v.mid.is_zero())
                    dot_accumulate_radius(a, mag_upper_from_apfloat(v.mid), u.rad, plan.e_rad);
                if (!u.rad.is_zero() && !v.rad.is_zero())
                    dot_accumulate_radius(a, u.rad, v.rad, plan.e_rad);
            }
            s.err = a.err;
            s.srad = a.srad;
            if (acc)
                for (size_t l = 0; l < plan.n_s && int64_t(l) < acc_stride; l++)
                    acc[b * acc_stride + int64_t(l)] = a.s[l];
        }
        dot_tuning().disable_precision_reduction = false;
    });
}

// dot_complex_ball / dot_complex_approx (src/dot.cpp:549-568)
int ref_dot_complex_batch(const apb_balls* xre, const apb_balls* xim, const apb_balls* yre,
                          const apb_balls* yim, const apb_dot_index* ix, int64_t n, int64_t batch,
                          int64_t prec, int mode, int force_threeprod, apb_balls* ore,
                          apb_balls* oim, uint64_t* hits, int threads) {
    dot_threeprod_hits() = 0;  // thread-local counter of the calling thread (threads == 1 for counts)
    return guarded([&] {
        parallel_for(batch, threads, [&](int64_t lo, int64_t hi) {
            dot_tuning().force_threeprod = force_threeprod != 0;
            std::vector<ComplexBall> xs(static_cast<size_t>(n)), ys(static_cast<size_t>(n));
            for (int64_t b = lo; b < hi; b++) {
                for (int64_t i = 0; i < n; i++) {
                    int64_t ex = x_elem(ix, b, i), ey = y_elem(ix, b, i);
                    xs[size_t(i)] = {load_ball(xre, ex), load_ball(xim, ex)};
                    ys[size_t(i)] = {load_ball(yre, ey), load_ball(yim, ey)};
                }
                if (mode == APB_DOT_APPROX) {
                    ApComplex r = dot_complex_approx(xs.data(), 1, ys.data(), 1, size_t(n), prec);
                    store_ball(ore, b, Ball::exact(r.re));
                    store_ball(oim, b, Ball::exact(r.im));
                } else {
                    ComplexBall r = dot_complex_ball(xs.data(), 1, ys.data(), 1, size_t(n), prec);
                    store_ball(ore, b, r.re);
                    store_ball(oim, b, r.im);
                }
            }
            dot_tuning().force_threeprod = false;
        });
        if (hits) *hits = dot_threeprod_hits();
    });
}

// matmul_auto / block_matmul_ball / classical_matmul_ball (src/matmul.cpp:442-531).
// threads > 1 splits A into row blocks (bit-identical for single-block plans,
// SURVEY.md 8d); stats receives block count etc. of the (last) call.
int ref_matmul(const apb_mat* A, const apb_mat* B, int64_t prec, int algo, apb_mat* C,
               int threads, apb_matmul_stats* stats) {
    return guarded([&] {
        BallMatrix a = load_matrix(A), b = load_matrix(B);
        auto run = [&](const BallMatrix& aa) {
            if (algo == APB_MM_BLOCK) return block_matmul_ball(aa, b, prec);
            if (algo == APB_MM_CLASSICAL) return classical_matmul_ball(aa, b, prec);
            return matmul_auto(aa, b, prec);
        };
        matmul_stats().reset();
        if (threads <= 1) {
            BallMatrix c = run(a);
            store_matrix(C, c);
        } else {
            const int64_t m = A->rows;
            parallel_for(m, threads, [&](int64_t lo, int64_t hi) {
                BallMatrix part(static_cast<size_t>(hi - lo), a.cols);
                for (int64_t i = lo; i < hi; i++)
                    for (size_t j = 0; j < a.cols; j++) part.at(size_t(i - lo), j) = a.at(size_t(i), j);
                BallMatrix c = run(part);
                for (int64_t i = lo; i < hi; i++)
                    for (size_t j = 0; j < c.cols; j++)
                        store_ball(&C->b, i * C->cols + int64_t(j), c.at(size_t(i - lo), j));
            });
        }
        if (stats) {
            std::memset(stats, 0, sizeof *stats);
            stats->classical_calls = matmul_stats().classical_calls;
            stats->block_calls = matmul_stats().block_calls;
            stats->int_gemm_products = matmul_stats().multimod_products;
            stats->last_block_count = matmul_stats().last_block_count;
        }
    });
}

int ref_matmul_complex(const apb_mat* Are, const apb_mat* Aim, const apb_mat* Bre,
                       const apb_mat* Bim, int64_t prec, apb_mat* Cre, apb_mat* Cim, int threads) {
    return guarded([&] {
        BallMatrix ar = load_matrix(Are), ai = load_matrix(Aim);
        BallMatrix br = load_matrix(Bre), bi = load_matrix(Bim);
        ComplexBallMatrix b = ComplexBallMatrix::from_parts(br, bi);
        const int64_t m = Are->rows;
        parallel_for(m, threads, [&](int64_t lo, int64_t hi) {
            BallMatrix pr(static_cast<size_t>(hi - lo), ar.cols), pi(static_cast<size_t>(hi - lo), ar.cols);
            for (int64_t i = lo; i < hi; i++)
                for (size_t j = 0; j < ar.cols; j++) {
                    pr.at(size_t(i - lo), j) = ar.at(size_t(i), j);
                    pi.at(size_t(i - lo), j) = ai.at(size_t(i), j);
                }
            ComplexBallMatrix c = complex_matmul_ball(ComplexBallMatrix::from_parts(pr, pi), b, prec);
            for (int64_t i = lo; i < hi; i++)
                for (size_t j = 0; j < c.cols; j++) {
                    store_ball(&Cre->b, i * Cre->cols + int64_t(j), c.at(size_t(i - lo), j).re);
                    store_ball(&Cim->b, i * Cim->cols + int64_t(j), c.at(size_t(i - lo), j).im);
                }
        });
    });
}

// plan_blocks (src/matmul.cpp:132-161): (lo, hi, basecase) triples
int ref_plan_blocks(const apb_mat* A, const apb_mat* B, int64_t prec, int64_t* steps,
                    int64_t max_steps, int64_t* n_steps, int64_t* entry_prec_ab) {
    return guarded([&] {
        BallMatrix a = load_matrix(A), b = load_matrix(B);
        auto st = plan_blocks(a, b, prec);
        *n_steps = int64_t(st.size());
        for (size_t i = 0; i < st.size() && int64_t(i) < max_steps; i++) {
            steps[3 * i] = int64_t(st[i].lo);
            steps[3 * i + 1] = int64_t(st[i].hi);
            steps[3 * i + 2] = st[i].basecase ? 1 : 0;
        }
        if (entry_prec_ab) {
            entry_prec_ab[0] = entry_precision(a);
            entry_prec_ab[1] = entry_precision(b);
        }
    });
}

// int_matmul(scale_block_rows(A), scale_block_cols(B)) (include/apball/matmul.hpp:77-84):
// exact product as two's complement limbs, out_limbs per entry.
int ref_block_int_product(const apb_mat* A, const apb_mat* B, int64_t lo, int64_t hi,
                          int64_t* row_scale, int64_t* col_scale, uint64_t* out, int64_t out_limbs,
                          int64_t* heights) {
    return guarded([&] {
        BallMatrix a = load_matrix(A), b = load_matrix(B);
        std::vector<int64_t> ei, fj;
        IntMatrix ia = scale_block_rows(a, size_t(lo), size_t(hi), ei);
        IntMatrix ib = scale_block_cols(b, size_t(lo), size_t(hi), fj);
        if (heights) {
            heights[0] = int64_t(ia.height());
            heights[1] = int64_t(ib.height());
        }
        IntMatrix t = int_matmul(ia, ib, IntMulAlgo::Auto);
        for (size_t i = 0; i < ei.size(); i++) row_scale[i] = ei[i];
        for (size_t j = 0; j < fj.size(); j++) col_scale[j] = fj[j];
        for (size_t e = 0; e < t.a.size(); e++) {
            uint64_t* dst = out + int64_t(e) * out_limbs;
            std::memset(dst, 0, sizeof(uint64_t) * size_t(out_limbs));
            const BigInt& v = t.a[e];
            auto l = v.limbs();
            if (int64_t(l.size()) > out_limbs ||
                (int64_t(l.size()) == out_limbs && (l.back() >> 63)))
                throw std::length_error("ref_block_int_product: out_limbs too small");
            for (size_t k = 0; k < l.size(); k++) dst[k] = l[k];
            if (v.negative()) {  // two's complement negate
                uint64_t carry = 1;
                for (int64_t k = 0; k < out_limbs; k++) {
                    uint64_t w = ~dst[k] + carry;
                    carry = (carry && w == 0) ? 1 : 0;
                    dst[k] = w;
                }
            }
        }
    });
}

// radius_matmul_upper (src/matmul.cpp:368-438)
int ref_radius_matmul_upper(const uint32_t* pm, const int64_t* pe, const uint32_t* qm,
                            const int64_t* qe, int64_t m, int64_t n, int64_t k, uint32_t* om,
                            int64_t* oe) {
    return guarded([&] {
        MagMatrix p = load_mags(pm, pe, m, n), q = load_mags(qm, qe, n, k);
        MagMatrix c = radius_matmul_upper(p, q);
        for (int64_t i = 0; i < m * k; i++) {
            const Mag& r = c.a[size_t(i)];
            om[i] = r.is_zero() ? 0 : (r.is_inf() ? APB_RAD_INF : uint32_t(r.mantissa()));
            oe[i] = r.is_zero() || r.is_inf() ? 0 : r.exponent();
        }
    });
}

// oracle containment: the exact interval hull of initial + (-1)^sub sum x_i y_i
// (oracle::interval_dot_hull, src/oracle.cpp:489-506) inside the output ball.
// ok[b] = 1 contained, 0 not contained.
int ref_dot_contains(const apb_balls* x, const apb_balls* y, const apb_balls* initial,
                     int subtract, const apb_dot_index* ix, int64_t n, int64_t batch,
                     const apb_balls* out, uint8_t* ok, int threads) {
    return guarded([&] {
        parallel_for(batch, threads, [&](int64_t lo, int64_t hi) {
            std::vector<Ball> xs(static_cast<size_t>(n)), ys(static_cast<size_t>(n));
            for (int64_t b = lo; b < hi; b++) {
                for (int64_t i = 0; i < n; i++) {
                    xs[size_t(i)] = load_ball(x, x_elem(ix, b, i));
                    Ball yy = load_ball(y, y_elem(ix, b, i));
                    ys[size_t(i)] = subtract ? yy.neg() : yy;
                }
                Ball res = load_ball(out, b);
                if (res.mid.is_nan() || res.rad.is_inf()) {
                    ok[b] = 1;
                    continue;
                }
                oracle::RationalInterval hull =
                    oracle::interval_dot_hull({xs.data(), size_t(n)}, {ys.data(), size_t(n)});
                if (initial) {
                    oracle::RationalInterval ii = oracle::interval_from_ball(load_ball(initial, b));
                    hull.lo = hull.lo + ii.lo;
                    hull.hi = hull.hi + ii.hi;
                }
                oracle::RationalInterval r = oracle::interval_from_ball(res);
                ok[b] = (r.lo <= hull.lo && hull.hi <= r.hi) ? 1 : 0;
            }
        });
    });
}

// |a - b| <= 2^e_tol * S style check helper: exact sum |x_i y_i| as a Mag upper bound
// (used for the "midpoint within 2^-p sum|xy|" criterion).
int ref_abs_dot_upper(const apb_balls* x, const apb_balls* y, const apb_dot_index* ix, int64_t n,
                      int64_t batch, uint32_t* man, int64_t* ex) {
    return guarded([&] {
        for (int64_t b = 0; b < batch; b++) {
            oracle::Dyadic s;
            for (int64_t i = 0; i < n; i++) {
                ApFloat xm = load_mid(x, x_elem(ix, b, i)), ym = load_mid(y, y_elem(ix, b, i));
                if (xm.is_zero() || ym.is_zero()) continue;
                s = s + (oracle::dyadic_from_apfloat(xm) * oracle::dyadic_from_apfloat(ym)).abs();
            }
            if (s.is_zero()) {
                man[b] = 0;
                ex[b] = 0;
                continue;
            }
            auto limbs = s.m.to_limbs64();
            Mag mg = Mag::from_limbs_upper({limbs.data(), limbs.size()}, s.e);
            man[b] = uint32_t(mg.mantissa());
            ex[b] = mg.exponent();
        }
    });
}

// elementwise ball_add / ball_sub (src/ball.cpp:15-19, include/apball/ball.hpp:50-52)
int ref_ball_addsub(const apb_balls* x, const apb_balls* y, int subtract, int64_t count, int64_t prec,
                    apb_balls* out) {
    return guarded([&] {
        for (int64_t i = 0; i < count; i++) {
            Ball a = load_ball(x, i), b = load_ball(y, i);
            store_ball(out, i, subtract ? ball_sub(a, b, prec) : ball_add(a, b, prec));
        }
    });
}

// the reference's own verify suites (src/bench.cpp:486-731), for pinning
// poly_mullow_classical / series_exp_basecase (include/apball/poly.hpp:23-29)
int ref_poly_mullow(const apb_balls* a, int64_t alen, const apb_balls* b, int64_t blen, int64_t len,
                    int64_t prec, apb_balls* out) {
    return guarded([&] {
        BallPoly pa, pb;
        for (int64_t i = 0; i < alen; i++) pa.c.push_back(load_ball(a, i));
        for (int64_t i = 0; i < blen; i++) pb.c.push_back(load_ball(b, i));
        BallPoly r = poly_mullow_classical(pa, pb, size_t(len), prec);
        for (int64_t k = 0; k < len; k++) store_ball(out, k, r.c[size_t(k)]);
    });
}

int ref_series_exp(const apb_balls* a, int64_t alen, int64_t len, int64_t prec, apb_balls* out) {
    return guarded([&] {
        BallPoly pa;
        for (int64_t i = 0; i < alen; i++) pa.c.push_back(load_ball(a, i));
        BallPoly r = series_exp_basecase(pa, size_t(len), prec);
        for (int64_t k = 0; k < len; k++) store_ball(out, k, r.c[size_t(k)]);
    });
}

// Ball::to_string / Ball::parse (src/ball.cpp:45-56): the reference's text form
int64_t ref_balls_format(const apb_balls* a, int64_t first, int64_t count, char* buf, int64_t cap) {
    std::string s;
    for (int64_t i = first; i < first + count; i++) s += load_ball(a, i).to_string() + "\n";
    const int64_t n = (int64_t)s.size();
    if (buf && cap > n) {
        std::memcpy(buf, s.data(), size_t(n));
        buf[n] = 0;
    }
    return n;
}

int64_t ref_balls_parse(const char* text, int64_t len, apb_balls* out, int64_t count) {
    std::string_view v(text, size_t(len));
    int64_t i = 0;
    while (i < count && !v.empty()) {
        auto nl = v.find('\n');
        auto b = Ball::parse(v.substr(0, nl));
        if (!b) return -1;
        store_ball(out, i++, *b);
        v = nl == std::string_view::npos ? std::string_view() : v.substr(nl + 1);
    }
    return i;
}

int ref_run_verify_suite(const char* name, uint64_t trials, uint64_t seed, uint64_t* failures) {
    return guarded([&] {
        std::string s(name);
        bench::VerifyReport r;
        if (s == "dot_containment") r = bench::verify_dot_containment(trials, seed);
        else if (s == "dot_exact_zero") r = bench::verify_dot_exact_zero(trials, seed);
        else if (s == "dot_accuracy") r = bench::verify_dot_accuracy_bound(trials, seed);
        else if (s == "matmul_block_accuracy") r = bench::verify_matmul_block_accuracy(trials, seed);
        else if (s == "matmul_planner") r = bench::verify_matmul_planner();
        else throw std::invalid_argument("unknown suite");
        *failures = r.failures;
    });
}

}  // extern "C"
