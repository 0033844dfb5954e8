"""Load the golden fixtures written by oracle/gen_golden.py."""
import glob
import os

import numpy as np

from paper_1901_04289_b200.balls import BallArray, apb_dot_index

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def files(prefix):
    return sorted(glob.glob(os.path.join(GOLDEN, prefix + "*.npz")))


def balls(d, prefix):
    if f"{prefix}_mant" not in d:
        return None
    return BallArray(d[f"{prefix}_mant"], d[f"{prefix}_exp"], d[f"{prefix}_kind"],
                     d[f"{prefix}_rad_man"], d[f"{prefix}_rad_exp"])


def index(d):
    v = [int(t) for t in d["idx"]]
    return apb_dot_index(*v)


def name(path):
    return os.path.basename(path)[:-4]
