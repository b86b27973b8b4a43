"""Trace rendering of device-produced OutRecords: the lines rendered
from the GPU's records equal those rendered from the oracle's (the renderer itself is pinned
against the reference in tests/test_trace_format.py), and a dumped buffer replays on the GPU."""

import numpy as np
import pytest

from paper_2605_26461_b200 import synth
from paper_2605_26461_b200 import tracefmt as T
from paper_2605_26461_b200.engine import BatchParams, FaultEngine

from oracle import seq_oracle as so

pytestmark = pytest.mark.gpu


def test_gpu_records_render_like_oracle(tmp_path):
    w, trace = synth.make_config("c2b", n=200_000)
    eng = FaultEngine(0)
    eng.upload_world(w)
    for iso in (True, False):
        got = eng.process(trace, BatchParams(isolation=iso))
        want = so.process_batch(w, trace, so.Params(isolation=iso))
        a = T.render_trace(trace, got.out, w.channel_names, w.client_names, t_drain=11)
        b = T.render_trace(trace, want.out, w.channel_names, w.client_names, t_drain=11)
        assert a == b and len(a) > 0
    path = str(tmp_path / "c2b.mpsfbuf")
    T.write_dump(path, trace, w.channel_names, w.client_names, isolation=True)
    d = T.read_dump(path)
    r = eng.process(np.asarray(d.entries), BatchParams(isolation=d.isolation))
    assert np.array_equal(r.out, eng.process(trace, BatchParams(isolation=True)).out)
    eng.close()
