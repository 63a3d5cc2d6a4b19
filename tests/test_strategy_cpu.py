"""CPU: the block-size strategy (decide) — oracle and the product's host state
machine (bk_host_decide_sequence) against the reference's exact decision
sequences (proj/tests/test_strategy.cpp:72-209), then against each other on
random residual histories."""
import ctypes as C
import json
import os

import numpy as np
import pytest

from paper_2409_05572_b200 import blockeig as B
from tests.oracle_api import OracleKernels

KA = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_known_answers.json")))
SEQ = KA["strategy_sequences"]
KINDS = {"none": 0, "fix": 1, "slope": 2, "slopek": 3}


class ProductStrategy:
    def __init__(self, path):
        self.f = C.CDLL(path).bk_host_decide_sequence
        self.f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_double,
                           C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                           C.POINTER(C.c_int)]

    def run(self, s, r, n_es, n_ex, start_n_now, start_shrunk, apply=True):
        r = np.ascontiguousarray(r, dtype=np.float64)
        out = np.zeros(len(r), dtype=np.int32)
        code = self.f(s.kind, s.j_e, s.j_s, s.mu, s.j_p, s.j_warm, s.r_warm, r.ctypes.data_as(C.POINTER(C.c_double)),
                      len(r), n_es, n_ex, start_n_now, int(start_shrunk), int(apply), out.ctypes.data_as(C.POINTER(C.c_int)))
        assert code == 0
        return list(out)


@pytest.fixture(scope="module")
def both(oracle, product_path):
    ok = OracleKernels(oracle)
    ps = ProductStrategy(product_path)
    def orc(s, r, n_es, n_ex, start_n_now, start_shrunk, apply=True):
        return ok.decide_sequence(s, r, n_es, n_ex, start_n_now, start_shrunk, apply_changes=apply)[0]
    return [("oracle", orc), ("product", ps.run)], ok


def strat(oracle, kind, **kw):
    return oracle.strategy_config(kind, **kw)


def test_slope_helpers(oracle):
    ok = OracleKernels(oracle)
    for lr, want in KA["slope_helpers"]["slope"]:
        assert ok.slope(lr) == pytest.approx(want)
    for lr, jp, want in KA["slope_helpers"]["slope_avg"]:
        assert ok.slope(lr, jp) == pytest.approx(want)


def test_reference_sequences(oracle, both):
    runners, ok = both
    es, ex = SEQ["n_es"], SEQ["n_ex"]
    w = SEQ["warmup"]
    s = strat(oracle, "fix", j_warm=w["j_warm"], r_warm=w["r_warm"])
    f = SEQ["fix_period"]
    sf = strat(oracle, "fix", j_e=f["j_e"], j_s=f["j_s"], j_warm=f["j_warm"], r_warm=f["r_warm"])
    sl = SEQ["slope"]
    ss = strat(oracle, "slope", mu=sl["mu"])
    st = SEQ["slope_stall"]
    sk = SEQ["slopek_window"]
    sks = strat(oracle, "slopek", j_p=sk["j_p"])
    for name, run in runners:
        assert run(s, w["r"], es, ex, w["start_n_now"], w["start_shrunk"]) == w["want"], name
        assert run(sf, [f["r_const"]] * len(f["want"]), es, ex, f["start_n_now"], f["start_shrunk"]) == f["want"], name
        assert run(ss, 10.0 ** np.array(sl["log10_r"]), es, ex, sl["start_n_now"], sl["start_shrunk"]) == sl["want"], name
        assert run(strat(oracle, "slope"), 10.0 ** np.array(st["log10_r"]), es, ex, 10, 1) == st["want"], name
        r = 10.0 ** (sk["log10_r_slope"] * np.arange(1, sk["count"] + 1))
        assert run(sks, r, es, ex, 10, 1) == [0] * sk["count"], name
    # c_max reset after the shrink (test_strategy.cpp:111-129)
    _, cmax = ok.decide_sequence(ss, 10.0 ** np.array(sl["log10_r"]), es, ex, 10, 1)
    assert cmax == pytest.approx(sl["c_max_after"])


def test_between_targets_holds(oracle, both):
    runners, _ = both
    for name, run in runners:
        d = run(strat(oracle, "slope"), 10.0 ** (-0.5 * np.arange(20)), 10, 20, 15, 1, apply=False)
        assert d == [0] * 20, name


def test_oscillation(oracle, both):
    runners, _ = both
    j = np.arange(1, 41)
    r = 10.0 ** (-0.1 * j + 0.15 * np.where(j % 2 == 1, -1, 1))
    for name, run in runners:
        d1 = run(strat(oracle, "slope", mu=1.1, j_p=10), r, 10, 20, 10, 1)
        d2 = run(strat(oracle, "slopek", mu=1.1, j_p=10), r, 10, 20, 10, 1)
        assert d1.count(2) >= 1 and d2.count(2) == 0, name


def test_shrink_lags_expand(oracle, both):
    runners, _ = both
    j = np.arange(1, 61)
    r = 10.0 ** (-0.2 * j + np.where(j % 7 == 0, 0.8, 0.0))
    for kind in ("fix", "slope", "slopek"):
        s = strat(oracle, kind, j_e=5, j_s=2, j_p=2, j_warm=0, r_warm=1.0)
        for name, run in runners:
            d = run(s, r, 10, 20, 20, 0)
            last = -1
            assert d.count(2) >= 1
            for i, x in enumerate(d, start=1):
                if x == 2:
                    last = i
                if x == 1 and last >= 0:
                    assert i - last == 2, (name, kind)


@pytest.mark.parametrize("seed", range(8))
def test_product_matches_oracle_random(oracle, both, seed):
    runners, _ = both
    rng = np.random.default_rng(seed)
    r = 10.0 ** np.cumsum(rng.normal(-0.1, 0.3, 200))
    for kind in ("none", "fix", "slope", "slopek"):
        s = strat(oracle, kind, j_e=int(rng.integers(3, 15)), j_s=2, mu=float(rng.uniform(1.0, 1.5)),
                  j_p=int(rng.integers(1, 12)), j_warm=int(rng.integers(0, 8)), r_warm=float(10 ** rng.uniform(-6, 0)))
        outs = [run(s, r, 10, 20, 20, 0) for _, run in runners]
        assert outs[0] == outs[1], kind


def test_normal_stream_bit_identical(oracle, product_path):
    # the product's background normal stream == std::normal_distribution per
    # block over one std::mt19937_64 (reference random_block, kernel.cpp:166-172),
    # including the discarded cached value after odd-sized blocks
    sizes = np.array([7, 1, 64, 33, 2, 5000, 3], dtype=np.int32)
    total = int(sizes.sum())
    got = np.zeros(total)
    want = np.zeros(total)
    pf = C.CDLL(product_path).bk_host_normal_blocks
    pf.argtypes = [C.c_uint64, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double)]
    assert pf(11, sizes.ctypes.data_as(C.POINTER(C.c_int)), len(sizes), got.ctypes.data_as(C.POINTER(C.c_double))) == 0
    of = oracle.lib.orc_random_blocks
    of.argtypes = [C.c_uint64, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_double)]
    of(11, sizes.ctypes.data_as(C.POINTER(C.c_int)), len(sizes), want.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(got, want)
