"""GPU: the Dataset path (d2ft_engine_step_units) — the trainer's batch body
fed from the reference's fp64 vector<Matrix> (data.hpp:18-42,
trainer.cpp:247-253), gathered H2D and converted on the device.  It must give
the same bytes as the fp32 host-buffer path (d2ft_engine_step) on the same
batch, with and without the next-batch prefetch, and reject what the
reference rejects."""
import numpy as np
import pytest

import paper_2504_12471_b200 as P
from paper_2504_12471_b200 import engine as E
from oracle import lib as O

pytestmark = pytest.mark.gpu

CFG = E.ModelConfig(2, 2, 128, 256, 50, 4, 5)  # dh = 64 (tcgen05 attention), ragged T


def _setup(n_samples=16, mbs=1, seed=4):
    ds = E.make_synthetic_dataset_f64(n_samples, CFG.num_classes, CFG.model_dim, CFG.seq_len, 0.5, 7)
    K = CFG.scheduled_subnet_count()
    units = ds.micro_batch_count(mbs)
    b, f = O.bench_scores(K, units, seed)
    scores = P.ScoreTable(K, units, f, b)
    return ds, scores


def _slice(scores, units):
    return P.ScoreTable(scores.subnets, len(units), scores.forward[:, units], scores.backward[:, units])


@pytest.mark.parametrize("mbs", [1, 2])
def test_step_units_equals_host_buffer_step(mbs):
    ds, scores = _setup(16, mbs)
    K = CFG.scheduled_subnet_count()
    rng = np.random.default_rng(11)
    order = rng.permutation(ds.micro_batch_count(mbs)).astype(np.int32)
    n_mb = 4
    caps = P.Capacities([(2 * n_mb // 5 + 1) * 5] * K, [(2 * n_mb // 5) * 2] * K)
    a = E.SubnetModel(CFG, n_mb * mbs)
    b = E.SubnetModel(CFG, n_mb * mbs)
    c = E.SubnetModel(CFG, n_mb * mbs)
    batches = [order[i * n_mb:(i + 1) * n_mb] for i in range(len(order) // n_mb)]
    for i, units in enumerate(batches):
        nxt = batches[i + 1] if i + 1 < len(batches) else None
        la, ta = a.step_units(ds, units, scores, P.CostModel(), caps, mbs, 0.05, 0.9, units_next=nxt)
        lc, tc = c.step_units(ds, units, scores, P.CostModel(), caps, mbs, 0.05, 0.9)  # no prefetch
        x = np.stack([s for u in units for s in ds.unit_inputs(int(u), mbs)]).astype(np.float32)
        y = np.concatenate([ds.unit_labels(int(u), mbs) for u in units])
        lb, tb = b.d2ft_step(x, y, _slice(scores, units), P.CostModel(), caps, mbs, 0.05, 0.9)
        assert np.array_equal(ta.codes, tb.codes) and np.array_equal(tc.codes, tb.codes)
        ref = O.knapsack_schedule(scores.backward[:, units], scores.forward[:, units], 2, 3, caps.full, caps.fwd)
        assert np.array_equal(ta.codes, ref)
        assert la == lb == lc
    pa, pb, pc = a.params(), b.params(), c.params()
    assert np.array_equal(pa, pb) and np.array_equal(pc, pb)
    assert np.array_equal(a.velocity(), b.velocity())
    for m in (a, b, c):
        m.close()
    ds.close()


def test_step_units_errors():
    ds, scores = _setup(8, 1)
    K = CFG.scheduled_subnet_count()
    caps = P.Capacities([10] * K, [4] * K)
    m = E.SubnetModel(CFG, 4)
    p0 = m.params()
    with pytest.raises(E.Error) as e:
        m.step_units(ds, [0, 1, 2, 99], scores, P.CostModel(), caps)
    assert e.value.kind == "input"
    with pytest.raises(E.Error) as e:  # the table must cover every unit of the dataset
        m.step_units(ds, [0, 1, 2, 3], _slice(scores, [0, 1, 2, 3]), P.CostModel(), caps)
    assert e.value.kind == "input"
    with pytest.raises(E.Error) as e:
        m.step_units(ds, [0, 1, 2, 3, 4], scores, P.CostModel(), P.Capacities([10] * K, [4] * K))
    assert e.value.kind == "size"
    bad = P.ScoreTable(K, 8, scores.forward.copy(), scores.backward.copy())
    bad.forward[0, 2] = np.nan  # unit 2 is in the batch: its slice carries the NaN
    with pytest.raises(E.Error) as e:
        m.step_units(ds, [0, 1, 2, 3], bad, P.CostModel(), caps)
    assert e.value.kind == "numeric"
    assert np.array_equal(m.params(), p0)  # nothing ran
    # a prefetch of other units must not be consumed silently
    m.step_units(ds, [0, 1, 2, 3], scores, P.CostModel(), caps, units_next=[4, 5, 6, 7])
    with pytest.raises(E.Error) as e:
        m.step_units(ds, [7, 6, 5, 4], scores, P.CostModel(), caps)
    assert e.value.kind == "state"
    m.step_units(ds, [4, 5, 6, 7], scores, P.CostModel(), caps)
    m.close()
    ds.close()


def test_step_units_unaligned_heap_samples():
    """Samples sharing pages (small heap matrices) cannot all be page-locked;
    the gather still reads the right bytes."""
    ds0, scores = _setup(8, 1)
    flat = np.stack(ds0.samples)
    big = np.empty(flat.size + 3, np.float64)[3:].reshape(flat.shape)  # 24-byte offset, contiguous
    big[...] = flat
    ds = E.Dataset([big[i] for i in range(8)], ds0.labels, CFG.num_classes)
    K = CFG.scheduled_subnet_count()
    caps = P.Capacities([10] * K, [4] * K)
    a, b = E.SubnetModel(CFG, 4), E.SubnetModel(CFG, 4)
    la, _ = a.step_units(ds, [3, 1, 0, 6], scores, P.CostModel(), caps)
    lb, _ = b.step_units(ds0, [3, 1, 0, 6], scores, P.CostModel(), caps)
    assert la == lb and np.array_equal(a.params(), b.params())
    for x in (a, b, ds, ds0):
        x.close()


def test_step_units_staged_batch_follows_the_call():
    """units_next also stages the next batch's labels / score slice on the
    host; the next call uses that staging only for the same dataset, score
    table and cost / capacity rows — changed capacities or another score
    table give exactly the unstaged engine's step."""
    ds, scores = _setup(16, 1)
    _, scores2 = _setup(16, 1, seed=9)
    K = CFG.scheduled_subnet_count()
    n_mb = 4
    caps = P.Capacities([(2 * n_mb // 5 + 1) * 5] * K, [(2 * n_mb // 5) * 2] * K)
    caps2 = P.Capacities([5] * K, [2] * K)
    u0, u1, u2 = [0, 5, 2, 7], [1, 3, 4, 6], [8, 9, 10, 11]
    a = E.SubnetModel(CFG, n_mb)
    b = E.SubnetModel(CFG, n_mb)
    seq = [(u0, scores, caps, u1), (u1, scores, caps2, u2), (u2, scores2, caps, None)]
    for units, sc, cp, nxt in seq:
        la, ta = a.step_units(ds, units, sc, P.CostModel(), cp, 1, 0.05, 0.9, units_next=nxt)
        lb, tb = b.step_units(ds, units, sc, P.CostModel(), cp, 1, 0.05, 0.9)
        ref = O.knapsack_schedule(sc.backward[:, units], sc.forward[:, units], 2, 3, cp.full, cp.fwd)
        assert np.array_equal(ta.codes, ref) and np.array_equal(tb.codes, ref)
        assert la == lb
    assert np.array_equal(a.params(), b.params())
    for m in (a, b):
        m.close()
    ds.close()
