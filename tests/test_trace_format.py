"""Trace-line rendering (``mpsf_render_trace``) and the binary fault-buffer dump
(SURVEY.md §8(f) rank 4).

Rendering is host code in libmpsf.so (no device needed), so it is pinned here against the
reference itself: on random batches the reference processes (the [P11] method), the
reference's own trace lines of the top half (``fault_raised`` / ``shadow_copy``) and of the
drain (``bh_service`` / ``parse_fatal`` / ``tlb_invalidate`` / ``fatal_report`` /
``isolate_begin``) must equal the lines rendered from the batch's OutRecords (the oracle's,
which the GPU tests show are the device's bit for bit).  The dump tests round-trip a buffer
and replay it."""

import random

import numpy as np
import pytest

from paper_2605_26461_b200 import tracefmt as T
from paper_2605_26461_b200 import synth
from paper_2605_26461_b200.world import ENTRY_DTYPE, export_reference_world

from oracle import seq_oracle as so
from tests import refharness as H

TOP = {"fault_raised", "shadow_copy"}
DRAIN = {"bh_service", "parse_fatal", "tlb_invalidate", "fatal_report", "isolate_begin"}


def _reference_lines(w, flat, entries, isolation):
    """Run the batch through the reference; returns (top-half lines, drain lines) rendered by
    the reference's Trace, or None when the reference raises on the batch."""
    from mpssim import faults, pipeline
    from mpssim.execmodel import EngineClass
    from mpssim.kernel import Trace
    from mpssim.memory import AccessType, FaultSeed

    w.uvm.isolation_enabled = isolation
    for e in entries:
        ch = flat.channel_names[int(e["channel"])]
        kind = int(e["kind"])
        if kind == 0:
            pipeline.raise_mmu_fault(w, FaultSeed(va=int(e["va"]), access=AccessType(H.ACCESSES[int(e["access"])]),
                                                  engine=EngineClass(H.ENGINES[int(e["engine"])]), channel_id=ch))
        elif 1 <= kind <= 5:
            pipeline.raise_parse_time_fault(w, ch, faults.PARSE_TIME_ORDER[kind - 1])
    top_end = len(w.trace.records)
    try:
        for e in entries:
            if int(e["kind"]) >= 8:
                ch = flat.channel_names[int(e["channel"])]
                code = ("EXC_2", "EXC_4", "EXC_5", "EXC_6", "EXC_7")[int(e["kind"]) - 8]
                pipeline.raise_sm_trap(w, code, 0, w.gpu.channels[ch].owner_pid)
        drain_start = len(w.trace.records)
        pipeline.service_bottom_half(w)
    except Exception as exc:
        assert type(exc).__name__ in ("UnknownTsg", "KeyError"), repr(exc)
        return None
    recs = w.trace.records
    top = [Trace.render_record(r) for r in recs[:top_end] if r[2] in TOP]
    drain = [Trace.render_record(r) for r in recs[drain_start:] if r[2] in DRAIN]
    return top, drain


@pytest.mark.skipif(not H.reference_available(), reason="reference not present")
@pytest.mark.parametrize("seed", range(4))
def test_rendered_lines_equal_reference_trace(seed):
    H.import_reference()
    rnd = random.Random(4100 + seed)
    checked = 0
    for _ in range(40):
        spec = H.random_small_world_spec(rnd)
        params_kw = dict(m1_latency_us=rnd.choice((131, 300)), m2_latency_us=rnd.choice((2780, 100)),
                         m3_latency_us=rnd.choice((1700, 0)))
        w = H.build_reference_world(spec, params_kw)
        flat = export_reference_world(w)
        iso = rnd.random() < 0.6
        entries = H.random_batch(rnd, flat, rnd.randint(1, 12))
        p = so.Params(isolation=iso, benign_us=w.params.benign_service_us, m1_us=w.params.m1_latency_us,
                      m2_us=w.params.m2_latency_us, m3_us=w.params.m3_latency_us)
        res = so.process_batch(flat, entries, p)
        if np.any(res.out["verdict"] & 0x20):   # duplicates: the batch coalesces, the reference does not
            continue
        t = w.clock.now
        ref = _reference_lines(w, flat, entries, iso)
        if ref is None:
            continue
        m_us = (w.params.m1_latency_us, w.params.m2_latency_us, w.params.m3_latency_us)
        top = T.render_trace(entries, res.out, flat.channel_names, flat.client_names, t_drain=t,
                             parts=T.RENDER_TOP, m_us=m_us)
        drain = T.render_trace(entries, res.out, flat.channel_names, flat.client_names, t_drain=t,
                               parts=T.RENDER_DRAIN, m_us=m_us)
        assert top.splitlines() == ref[0]
        assert drain.splitlines() == ref[1]
        checked += 1
    assert checked >= 10


@pytest.mark.skipif(not H.reference_available(), reason="reference not present")
def test_rendered_lines_parse_with_reference_parser():
    H.import_reference()
    from mpssim.kernel import parse_trace_text
    w, trace = synth.make_config("c1", n=2000)
    res = so.process_batch(w, trace, so.Params(isolation=True))
    text = T.render_trace(trace, res.out, w.channel_names, w.client_names, t_drain=7)
    recs = list(parse_trace_text(text))
    assert recs and all(r["t"] == 7 for r in recs)
    assert sum(r["kind"] == "bh_service" for r in recs) == int(((trace["kind"] < 8) & (trace["flags"] & 1 != 0)).sum())


def test_render_threads_agree():
    w, trace = synth.make_config("c1", n=50_000)
    res = so.process_batch(w, trace, so.Params(isolation=True))
    one = T.render_trace(trace, res.out, w.channel_names, w.client_names, threads=1)
    many = T.render_trace(trace, res.out, w.channel_names, w.client_names, threads=8)
    assert one == many and one.endswith("\n")
    t_raise = np.arange(len(trace), dtype=np.uint64)
    top = T.render_trace(trace, res.out, w.channel_names, w.client_names, t_raise=t_raise, parts=T.RENDER_TOP)
    first = top.splitlines()[0]
    i0 = int(np.nonzero((trace["kind"] < 8) & (trace["flags"] & 1 != 0))[0][0])
    assert first.startswith(f"t={i0} ")


def test_render_empty_and_bad_args():
    e = np.zeros(0, ENTRY_DTYPE)
    from paper_2605_26461_b200.world import OUT_DTYPE
    assert T.render_trace(e, np.zeros(0, OUT_DTYPE), [], []) == ""
    with pytest.raises(ValueError):
        T.render_trace(np.zeros(2, ENTRY_DTYPE), np.zeros(1, OUT_DTYPE), [], [])


def test_dump_round_trip_and_replay(tmp_path):
    w, trace = synth.make_config("c1", n=10_000)
    t_raise = np.arange(len(trace), dtype=np.uint64) * 3
    path = str(tmp_path / "buf.mpsfbuf")
    T.write_dump(path, trace, w.channel_names, w.client_names, isolation=False, base_index=5, t_drain=99,
                 t_raise=t_raise)
    d = T.read_dump(path)
    assert np.array_equal(np.asarray(d.entries), trace)
    assert np.array_equal(np.asarray(d.t_raise), t_raise)
    assert d.channel_names == list(w.channel_names) and d.client_names == list(w.client_names)
    assert (d.isolation, d.base_index, d.t_drain) == (False, 5, 99)
    # replay: the dumped buffer processes and renders as the original
    a = so.process_batch(w, np.asarray(d.entries), so.Params(isolation=d.isolation))
    b = so.process_batch(w, trace, so.Params(isolation=False))
    assert np.array_equal(a.out, b.out)
    assert (T.render_trace(d.entries, a.out, d.channel_names, d.client_names, t_drain=d.t_drain, t_raise=d.t_raise)
            == T.render_trace(trace, b.out, w.channel_names, w.client_names, t_drain=99, t_raise=t_raise))
    # empty dump, no names, no raise times
    p2 = str(tmp_path / "empty.mpsfbuf")
    T.write_dump(p2, np.zeros(0, ENTRY_DTYPE))
    d2 = T.read_dump(p2)
    assert len(d2.entries) == 0 and d2.t_raise is None and d2.channel_names == []
    # not a dump
    p3 = tmp_path / "junk"
    p3.write_bytes(b"x" * 100)
    with pytest.raises(ValueError):
        T.read_dump(str(p3))
