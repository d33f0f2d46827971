"""Byte-for-byte parity of the artifact writers and readers (csrc/serialize.cu
through paper_2504_12471_b200/serialize.py) with the unmodified reference
serialize.cpp (compiled into oracle/_ref against the image's nlohmann json
3.11.3, oracle/Makefile).  CPU only; skipped where oracle/_ref is not built."""
import math
import re

import numpy as np
import pytest

from oracle import lib as O
from paper_2504_12471_b200 import cost_sim as CS
from paper_2504_12471_b200 import serialize as S
from paper_2504_12471_b200._lib import Error
from paper_2504_12471_b200.scheduler import ScheduleTable, ScoreTable

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def upstream_layout(text):
    """The only nlohmann json.hpp in this image (cudnn_frontend's copy of
    3.11.3, json.hpp:20610-20614, "Custom from FE") prints arrays whose first
    element is an integer on one line ("[1,3]"); upstream 3.11.3 — what the
    reference vendors — pretty-prints them like every other array.  The
    reference's integer arrays (schedule codes) are re-laid out upstream-style
    before comparing; every other byte is compared as produced."""
    out = []
    for line in text.split("\n"):
        m = re.fullmatch(r"( *)\[(-?\d+(?:,-?\d+)*)\](,?)", line)
        if not m:
            out.append(line)
            continue
        ind, body, comma = m.groups()
        vals = body.split(",")
        out.append(ind + "[")
        out += [ind + "  " + v + ("," if i + 1 < len(vals) else "") for i, v in enumerate(vals)]
        out.append(ind + "]" + comma)
    return "\n".join(out)


def _doubles(rng, n):
    """Awkward doubles: wide exponents, integral values, shortest-digit edge
    cases, subnormals, signed zero."""
    special = [0.0, -0.0, 1.0, 2.0, 0.1, 1 / 3, 1e-4, 1e-5, 9.999999999999999e-5, 1e14, 1e15, 1e16, 123456.789,
               5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 0.30000000000000004, 100.0, 1e21, 1e22,
               4.35, 2.675, 1e-7, 123e-20, -2.5e-7]
    rnd = list(rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n))
    rnd += list(np.round(rng.standard_normal(n) * 1000))
    return special + rnd


def test_format_double_bytes():
    rng = np.random.default_rng(1)
    for v in _doubles(rng, 300):
        assert S.format_double(v) == O.ref_format_double(v), v


def test_score_table_json_and_csv_bytes():
    rng = np.random.default_rng(2)
    vals = _doubles(rng, 100)
    for trial in range(30):
        K, N = int(rng.integers(0, 7)), int(rng.integers(0, 7))
        f = np.abs(np.array(rng.choice(vals, K * N) if K * N else [], np.float64)).reshape(K, N)
        b = np.abs(np.array(rng.choice(vals, K * N) if K * N else [], np.float64)).reshape(K, N)
        fm, bm = trial % 4, (trial * 3 + 1) % 4
        t = ScoreTable(K, N, f, b, S.METRICS[fm], S.METRICS[bm])
        assert S.score_table_to_json(t) == O.ref_score_table_text(f, b, fm, bm, 0)
        assert S.score_table_to_csv(t) == O.ref_score_table_text(f, b, fm, bm, 1)


def test_schedule_table_json_and_csv_bytes():
    rng = np.random.default_rng(3)
    for _ in range(30):
        K, N = int(rng.integers(0, 9)), int(rng.integers(0, 9))
        c = rng.integers(1, 4, (K, N)).astype(np.uint8)
        t = ScheduleTable(K, N, c)
        assert S.schedule_table_to_json(t) == upstream_layout(O.ref_schedule_table_text(c, 0))
        assert S.schedule_table_to_csv(t) == O.ref_schedule_table_text(c, 1)


def test_batch_metrics_bytes():
    rng = np.random.default_rng(4)
    vals = _doubles(rng, 50)
    for trial in range(30):
        m5 = [float(abs(x)) for x in rng.choice(vals, 5)]
        busy = [float(abs(x)) for x in rng.choice(vals, int(rng.integers(0, 9)))]
        run_id = ['r1', 'run "7"', 'a\\b', 'tab\there', 'unié', ''][trial % 6]
        method = ["d2ft", "random", "dpruning_mg", "moe"][trial % 4]
        m = CS.BatchMetrics(m5[0], m5[1], m5[2], m5[3], busy, m5[4])
        assert S.batch_metrics_to_json(m, run_id, method) == O.ref_batch_metrics_text(m5, busy, run_id, method, 0)
        assert S.batch_metrics_to_csv_row(m, run_id, method) == O.ref_batch_metrics_text(m5, busy, run_id, method, 1)
    assert S.batch_metrics_csv_header() == O.ref_batch_metrics_text([0] * 5, [], "", "", 2)


def test_history_bytes():
    rng = np.random.default_rng(5)
    vals = _doubles(rng, 50)
    for n in range(0, 8):
        eps = [(i, float(rng.choice(vals)), float(abs(rng.choice(vals))), float(rng.random()), float(rng.random()))
               for i in range(n)]
        h = S.TrainHistory([S.EpochRecord(*e) for e in eps])
        assert S.history_to_json(h) == O.ref_history_text(eps, 0)
        assert S.history_to_csv(h) == O.ref_history_text(eps, 1)


def test_readers_accept_what_the_reference_accepts():
    """Valid inputs (the reference's own writer output and hand-written
    variants: other key order, compact layout, integer-valued doubles,
    exponents, whitespace) parse to the same table as the reference."""
    score_docs = [
        '{"subnets":1,"micro_batches":2,"fwd_metric":"fisher_information","bwd_metric":"weight_magnitude",'
        '"forward":[[1,2.5]],"backward":[[0,3e-2]]}',
        '{ "backward": [ [ 1E2 , 0.0 ] ], "forward": [[0.25, 7]], "micro_batches": 2, "subnets": 1,'
        ' "bwd_metric": "taylor_importance", "fwd_metric": "gradient_magnitude" }',
        '{"subnets":0,"micro_batches":0,"fwd_metric":"fisher_information","bwd_metric":"weight_magnitude",'
        '"forward":[],"backward":[]}',
    ]
    for doc in score_docs:
        ours = S.score_table_from_json(doc)
        assert S.score_table_to_json(ours) == O.ref_reparse("score", doc)
    sched_docs = ['{"devices":2,"micro_batches":2,"codes":[[1,2],[3,1]]}',
                  '{ "codes" : [ [ 3 ] ], "micro_batches" : 1, "devices" : 1 }',
                  '{"devices":0,"micro_batches":0,"codes":[]}']
    for doc in sched_docs:
        assert S.schedule_table_to_json(S.schedule_table_from_json(doc)) == upstream_layout(O.ref_reparse("schedule", doc))
    hist_docs = ["epoch,loss,top1,compute_fraction,comm_fraction\n0,1.5,0.25,0.6,0.7\n1,0.5,0.5,0.6,0.7\n",
                 "any,header,is,skipped\n2,1.5,0.25,0.6,0.7\n\n",
                 "epoch,loss,top1,compute_fraction,comm_fraction\n1.9,2.5e3,0x1p-3,1,1,extra\n",
                 "epoch,loss,top1,compute_fraction,comm_fraction\n",
                 "epoch,loss,top1,compute_fraction,comm_fraction\n3,1e-05,1,0,0.5"]
    for doc in hist_docs:
        assert S.history_to_csv(S.history_from_csv(doc)) == O.ref_reparse("history", doc)


CATS = {1: "config", 2: "input", 3: "dimension", 4: "state", 5: "numeric", 6: "size"}


@pytest.mark.parametrize("kind,doc", [
    ("score", "not json"),
    ("score", '{"subnets":1}'),
    ("score", '{"subnets":"x","micro_batches":1,"fwd_metric":"fisher_information","bwd_metric":"weight_magnitude",'
              '"forward":[[1]],"backward":[[1]]}'),
    ("score", '{"subnets":1,"micro_batches":1,"fwd_metric":"nope","bwd_metric":"weight_magnitude",'
              '"forward":[[1]],"backward":[[1]]}'),
    ("score", '{"subnets":2,"micro_batches":1,"fwd_metric":"fisher_information","bwd_metric":"weight_magnitude",'
              '"forward":[[1]],"backward":[[1]]}'),
    ("score", '{"subnets":1,"micro_batches":1,"fwd_metric":"fisher_information","bwd_metric":"weight_magnitude",'
              '"forward":[[-1]],"backward":[[1]]}'),
    ("schedule", "[1,2]"),
    ("schedule", '{"devices":1,"micro_batches":1,"codes":[[4]]}'),
    ("schedule", '{"devices":1,"micro_batches":2,"codes":[[1]]}'),
    ("schedule", '{"devices":1,"micro_batches":1}'),
    ("history", "epoch,loss,top1,compute_fraction,comm_fraction\n1,2,3\n"),
    ("history", ""),
])
def test_readers_reject_like_the_reference(kind, doc):
    """Malformed inputs: same errc category and message as the reference."""
    with pytest.raises(O.OracleError) as r:
        O.ref_reparse(kind, doc)
    fn = {"score": S.score_table_from_json, "schedule": S.schedule_table_from_json,
          "history": S.history_from_csv}[kind]
    with pytest.raises(Error) as e:
        fn(doc)
    assert e.value.kind == CATS[r.value.code], (e.value, r.value)
    assert str(e.value).endswith(str(r.value).split(": ", 1)[-1]) or str(r.value) in str(e.value), (e.value, r.value)


def test_history_bad_field_is_an_input_error():
    """A non-numeric history field: the reference lets std::stoi's
    std::invalid_argument escape (not an errc category); the C-ABI cannot
    throw, so it reports an input error naming the field."""
    doc = "epoch,loss,top1,compute_fraction,comm_fraction\nx,1,1,1,1\n"
    with pytest.raises(O.OracleError) as r:
        O.ref_reparse("history", doc)
    assert r.value.code == 99 and "stoi" in str(r.value)
    with pytest.raises(Error) as e:
        S.history_from_csv(doc)
    assert e.value.kind == "input" and "'x'" in str(e.value)
