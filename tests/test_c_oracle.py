"""The C oracle (CPU baseline / fast checker) equals the Python oracle and the golden
fixtures; multi-threaded decode is deterministic."""

import random

import numpy as np

from paper_2605_26461_b200 import synth

from oracle import c_oracle as co
from oracle import seq_oracle as so
from tests import golden_io as G
from tests import randworld as RW
from tests.observe import observables


def same(a, b, ctx=""):
    for f in ("out", "verdict", "counts", "dedup_keys", "dedup_idx", "cancel"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), (ctx, f)


def test_c_oracle_equals_python_oracle_random():
    rnd = random.Random(99)
    for it in range(400):
        w = RW.random_world(rnd, dead_p=0.15 if it % 2 else 0.0)
        p = RW.random_params(rnd)
        e = RW.random_batch(rnd, w, rnd.randint(1, 80))
        same(co.process_batch(w, e, p), so.process_batch(w, e, p), it)


def test_c_oracle_golden_batches():
    for flat, entries, p, expect in G.batches():
        res = co.process_batch(flat, entries, so.Params(**p))
        assert observables(flat, entries, res.out, res.verdict) == G.as_tuples(expect)


def test_c_oracle_config1_threads():
    w, trace = synth.make_config("c1")
    a = co.process_batch(w, trace, so.Params(), threads=1)
    b = co.process_batch(w, trace, so.Params(), threads=8)
    same(a, b)
    c = so.process_batch(w, trace, so.Params())
    same(a, c)
