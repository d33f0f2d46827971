"""Generates the committed golden fixtures from the UNMODIFIED reference
(oracle/_ref/libd2ft_ref.so, built from /root/reference by oracle/Makefile).
Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py
Score tables are regenerated from (K, N, seed) with bench_scheduler.cpp's
make_scores recipe, so only codes, costs and capacities are stored."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import lib as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def schedules():
    d = {}

    def add(tag, K, N, seed, cf, cb, capf, capo):
        b, f = O.bench_scores(K, N, seed)
        cfa = np.full(K, cf, np.int32) if np.isscalar(cf) else np.asarray(cf, np.int32)
        cba = np.full(K, cb, np.int32) if np.isscalar(cb) else np.asarray(cb, np.int32)
        capf = np.asarray(np.broadcast_to(capf, (K,)), np.int32)
        capo = np.asarray(np.broadcast_to(capo, (K,)), np.int32)
        if np.all(cfa == cfa[0]) and np.all(cba == cba[0]):
            codes = O.ref_knapsack_schedule(b, f, int(cfa[0]), int(cba[0]), capf, capo, threads=8)
        else:
            codes = O.ref_knapsack_schedule(b, f, 0, 0, capf, capo, threads=8, cf_dev=cfa, cb_dev=cba)
        d["shape_" + tag] = np.array([K, N, seed], np.int64)
        d["cf_" + tag], d["cb_" + tag], d["capf_" + tag], d["capo_" + tag] = cfa, cba, capf, capo
        d["codes_" + tag] = codes

    # training shapes, budget floor(2N/5) p_f + floor(2N/5) p_o
    for tag, K, N in (("tiny", 8, 16), ("vitb", 144, 64), ("vitl", 384, 256)):
        nb = (2 * N) // 5
        add(tag, K, N, 1, 2, 3, nb * 5, nb * 2)
    # scheduler sweep 144 x 1024, r in {0.25, 0.5, 0.75, 1.0}
    for r in (0.25, 0.5, 0.75, 1.0):
        nr = int(r * 1024)
        add(f"sweep{int(r * 100)}", 144, 1024, 1, 2, 3, nr * 5, nr * 2)
    # heterogeneous per-device costs and capacities (cost_sim hetero profiles)
    rng = np.random.default_rng(5)
    add("hetero", 24, 48, 9, rng.integers(1, 4, 24), rng.integers(0, 5, 24), rng.integers(0, 200, 24),
        rng.integers(0, 60, 24))
    np.savez_compressed(os.path.join(OUT, "schedules.npz"), **d)


def dp():
    rng = np.random.default_rng(11)
    K, N = 12, 20
    scores = rng.random((K, N)) * 9.0
    weights = rng.integers(0, 8, (K, N)).astype(np.int32)
    weights[:4] = weights[:4, :1]  # some constant rows
    caps = rng.integers(0, 60, K).astype(np.int32)
    sel, obj = O.ref_dp_search(scores, weights, caps)
    np.savez_compressed(os.path.join(OUT, "dp_search.npz"), scores=scores, weights=weights, caps=caps, sel=sel,
                        obj=obj)


def rng_init():
    r = O.RefModel(2, 4, 32, 64, 16, 4, 1)
    x, y = O.ref_make_dataset(8, 4, 32, 16, 0.5, 7)
    np.savez_compressed(os.path.join(OUT, "rng_init.npz"), uniform_1_0=O.ref_uniform_stream(1, 0, 64),
                        shuffle_3_E000=O.ref_shuffle_iota(3, 0xE000, 40), params_tiny32=r.params(), data_x=x,
                        data_y=y)


def model_step():
    L, H, d, ffn, T, C = 2, 4, 32, 64, 16, 4
    r = O.RefModel(L, H, d, ffn, T, C, 1)
    rng = np.random.default_rng(3)
    p = r.params() + 0.05 * rng.standard_normal(r.n)  # nonzero biases exercise b1/b2 paths
    r.set_params(p)
    x, y = O.ref_make_dataset(4, C, d, T, 0.5, 7)
    codes = np.array([[1, 2, 3, 1], [2, 3, 1, 1], [3, 1, 2, 2], [1, 1, 1, 1],
                      [2, 2, 3, 1], [1, 3, 3, 2], [3, 3, 3, 3], [1, 2, 1, 3]], np.uint8)
    fb_loss, fb_grads, fb_eng = r.forward_backward(x[:2], y[:2], codes[:, 0])
    r2 = O.RefModel(L, H, d, ffn, T, C, 1)
    r2.set_params(p)
    loss = r2.train_batch(x, y, codes, 1, 0.05, 0.9)
    np.savez_compressed(os.path.join(OUT, "model_step.npz"), cfg=np.array([L, H, d, ffn, T, C]), params=p, x=x,
                        y=y, codes=codes, loss=loss, params_after=r2.params(), fb_grads=fb_grads,
                        fb_engaged=fb_eng)


if __name__ == "__main__":
    assert O.ref_available(), "build oracle/_ref first: make ref"
    schedules()
    dp()
    rng_init()
    model_step()
    print("golden fixtures written to", OUT)
