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
    {  // complex dots with the rewrite forced: identical results, hits counted
        DotTuning& tun = dot_tuning();
        tun.force_threeprod = true;
        const std::uint64_t h0 = dot_threeprod_hits();
        std::uint64_t ref_hits = 0, gpu_hits = 0;
        for (int t = 0; t < 20; t++) {
            std::vector<ComplexBall> x(9), y(9);
            for (auto& c : x) c = {Ball::exact(bench::random_apfloat(rng, 3, -80, 80)), Ball::exact(bench::random_apfloat(rng, 3, -80, 80))};
            for (auto& c : y) c = {Ball::exact(bench::random_apfloat(rng, 3, -80, 80)), Ball::exact(bench::random_apfloat(rng, 3, -80, 80))};
            const std::uint64_t a0 = dot_threeprod_hits();
            ComplexBall r = dot_complex_ball(x.data(), 1, y.data(), 1, 9, 1024);
            const std::uint64_t a1 = dot_threeprod_hits();
            ComplexBall g = b200::dot_complex_ball(x.data(), 1, y.data(), 1, 9, 1024);
            const std::uint64_t a2 = dot_threeprod_hits();
            ref_hits += a1 - a0;
            gpu_hits += a2 - a1;
            if (!complex_ball_identical(r, g)) bad++;
        }
        tun.force_threeprod = false;
        if (ref_hits != gpu_hits || ref_hits == 0) bad++;
        std::printf("threeprod hits ref %llu gpu %llu (start %llu)\n", (unsigned long long)ref_hits,
                    (unsigned long long)gpu_hits, (unsigned long long)h0);
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
