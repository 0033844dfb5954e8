"""The reference's text wire format in libapb_b200.so:
Ball::to_string / Ball::parse (src/ball.cpp:45-56, src/apfloat.cpp:333-390,
src/mag.cpp:174-197) and write/read_ball_matrix (src/matmul.cpp:552-570).
Host code -- these run without a GPU (the library loads on the CPU)."""
import numpy as np
import pytest

import pyoracle as po
from paper_1901_04289_b200 import _lib, gen, ops
from paper_1901_04289_b200.balls import BallArray


def _edge(seed, count, n):
    rng = np.random.Generator(np.random.PCG64(seed))
    x, y = gen.edge_dots(rng, count, n)
    return x.concat(y)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_format_matches_reference(seed):
    a = _edge(seed, 30, 11)  # limb counts 1-4, zeros, radii, +-inf, nan
    assert ops.balls_to_text(a) == po.balls_format(a)


@pytest.mark.parametrize("seed", [4, 5])
def test_round_trip_and_reference_parse(seed):
    a = _edge(seed, 25, 9)
    text = ops.balls_to_text(a)
    ours = ops.balls_from_text(text, a.count, a.L)
    theirs = po.balls_parse(text, a.count, a.L)
    assert ours.identical(a).all() and theirs.identical(a).all()


def test_kat_strings():
    one = BallArray.from_i64([1, -3, 0])
    assert ops.balls_to_text(one).splitlines() == [
        "(+,1,8000000000000000) +- 0", "(-,2,c000000000000000) +- 0", "0 +- 0"]


@pytest.mark.parametrize("bad", [
    "(+,1,4000000000000000) +- 0",                     # top bit not set (not normalized)
    "(+,1,8000000000000000:0000000000000000) +- 0",    # zero low limb (not minimal)
    "(+,1,800000000000000) +- 0",                      # 15 hex digits
    "(+,1,8000000000000000) +- (1000,3)",              # Mag mantissa outside [2^29, 2^30)
    "(+,1,8000000000000000) + 0",                      # missing " +- "
    "(*,1,8000000000000000) +- 0",                     # bad sign
])
def test_parse_rejects_malformed(bad):
    with pytest.raises(_lib.InvalidArgument):
        ops.balls_from_text(bad + "\n", 1, 2)
    assert po.balls_parse(bad + "\n", 1, 2) is None  # the reference rejects it too


def test_parse_rejects_too_wide_for_slots():
    a = BallArray.from_i64([1])
    wide = "(+,1,8000000000000000:0000000000000001:8000000000000000) +- 0\n"
    with pytest.raises(_lib.InvalidArgument):
        ops.balls_from_text(wide, 1, 2)
    assert ops.balls_from_text(wide, 1, 3).count == 1
    assert a.count == 1


def test_matrix_format_and_read():
    a = _edge(9, 4, 3)  # 24 balls -> a 4 x 6 matrix
    m = ops.BallMatrix(a, 4, 6)
    text = ops.matrix_to_text(m)
    assert text.startswith("4 6\n") and text[4:] == po.balls_format(a)
    back = ops.matrix_from_text(text, a.L)
    assert (back.rows, back.cols) == (4, 6) and back.balls.identical(a).all()
