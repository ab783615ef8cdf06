"""Adversarial inputs of tools/robust_time.py / one_build.py / knobs.py."""
import numpy as np

from paper_2211_00120_b200 import datagen

ADV = {
    "identical": lambda n, k: np.full((n, k), 0.25, np.float32),
    "huge": lambda n, k: (10.0 ** np.random.default_rng(4).uniform(-30, 30, (n, k))).astype(np.float32),
    "constaxis": lambda n, k: np.c_[datagen.uniform(n, k - 1, seed=3), np.zeros(n, np.float32)],
    "sorted": lambda n, k: np.sort(datagen.uniform(n, k, seed=2), axis=0),
    # float64 input (the reference's own dtype): the lbkd_build_*_f64 path
    "uniform64": lambda n, k: np.random.default_rng(0).random((n, k)),
}


def make(kind, n, k):
    return ADV[kind](n, k) if kind in ADV else datagen.make(kind, n, k, seed=0)
