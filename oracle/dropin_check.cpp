// TEST INFRASTRUCTURE: compiles include/apball_b200.hpp against the reference
// headers and runs the drop-in operators next to the reference ones on the
// same inputs (needs a GPU at run time).  Built by tests/test_dropin.py.
#include <cstdio>
#include <random>

#include "apball/bench.hpp"
#include "apball_b200.hpp"

using namespace apball;

int main() {
    bench::Rng rng(7);
    int bad = 0;
    for (int t = 0; t < 50; t++) {
        std::vector<Ball> x(37), y(37);
        for (auto& b : x) b = bench::random_ball(rng, 3, -40, 40, 50);
        for (auto& b : y) b = bench::random_ball(rng, 3, -40, 40, 50);
        Ball init = bench::random_ball(rng, 2, -40, 40, 50);
        Ball r = dot_ball(&init, t & 1, x.data() + 36, -1, y.data(), 1, 37, 130);
        Ball g = b200::dot_ball(&init, t & 1, x.data() + 36, -1, y.data(), 1, 37, 130);
        if (!ball_identical(r, g)) bad++;
    }
    BallMatrix a = bench::uniform_matrix(rng, 64, 192), b = bench::uniform_matrix(rng, 64, 192);
    BallMatrix c = block_matmul_ball(a, b, 192), g = b200::block_matmul_ball(a, b, 192);
    for (size_t i = 0; i < c.a.size(); i++)
        if (!ball_identical(c.a[i], g.a[i])) bad++;
    ComplexBallMatrix ca = ComplexBallMatrix::from_parts(a, b), cb = ComplexBallMatrix::from_parts(b, a);
    ComplexBallMatrix cc = complex_matmul_ball(ca, cb, 150), cg = b200::complex_matmul_ball(ca, cb, 150);
    for (size_t i = 0; i < cc.a.size(); i++)
        if (!complex_ball_identical(cc.a[i], cg.a[i])) bad++;
    for (int t = 0; t < 10; t++) {
        BallPoly pa, pb;
        for (int i = 0; i < 20 + t; i++) pa.c.push_back(bench::random_ball(rng, 2, -20, 20, 30));
        for (int i = 0; i < 15; i++) pb.c.push_back(bench::random_ball(rng, 2, -20, 20, 30));
        BallPoly r = poly_mullow_classical(pa, pb, 40, 128), g = b200::poly_mullow_classical(pa, pb, 40, 128);
        for (size_t k = 0; k < r.c.size(); k++)
            if (!ball_identical(r.c[k], g.c[k])) bad++;
        pa.c[0] = Ball::zero();
        BallPoly e = series_exp_basecase(pa, 12, 100), eg = b200::series_exp_basecase(pa, 12, 100);
        for (size_t k = 0; k < e.c.size(); k++)
            if (!ball_identical(e.c[k], eg.c[k])) bad++;
    }
    try {
        BallPoly one;
        one.c = {Ball::exact(ApFloat::from_i64(1))};
        b200::series_exp_basecase(one, 4, 64);
        bad++;
    } catch (const std::domain_error&) {
    }
    std::printf("dropin mismatches: %d\n", bad);
    return bad != 0;
}
