"""GPU results in the reference's text form: a device product written with
write_ball_matrix's format is byte-identical to the reference's own output
(the offline-diff use of the wire format)."""
import os

import pytest

import pyoracle as po
from paper_1901_04289_b200 import gen, ops

pytestmark = pytest.mark.gpu


def test_device_product_text_equals_reference_text():
    n, p = 96, 128
    a, b = gen.config2_matrices(n=n)
    got = ops.block_matmul_ball(ops.BallMatrix(a.to_device(), n, n), ops.BallMatrix(b.to_device(), n, n), p)
    ref, _ = po.matmul(a, b, n, n, n, p, which="ref", algo=1, threads=os.cpu_count() or 8)
    text = ops.matrix_to_text(got)
    assert text == f"{n} {n}\n" + po.balls_format(ref)
    back = ops.matrix_from_text(text, got.balls.L)
    assert back.balls.identical(ref).all()
