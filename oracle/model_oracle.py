"""ORACLE / TEST INFRASTRUCTURE ONLY — the CPU checker for the step numerics.

numpy fp64 restatement of the reference's subnet model, forward/backward and
trainer batch body.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg may import it; the product path never does.

Pinned against the unmodified reference (oracle/_ref/libd2ft_ref.so) to ~1e-12
relative in tests/test_oracle_vs_ref.py.

Parameters use the reference's canonical flat order (model.hpp:117-153):
  Embed: w_embed[d,d], b_embed[d], pos[T,d]
  Block(l,h) block-major/head-minor: wq,wk,wv[d,dh], wo[dh,d], w1[d,fs], b1[fs],
                                      w2[fs,d], b2[d/H]
  Head: w_cls[d,C], b_cls[C]
"""
from __future__ import annotations

from dataclasses import dataclass
import math

import numpy as np
from scipy.special import erf as _erf

LN_EPS = 1e-5  # model.hpp:32


@dataclass(frozen=True)
class Config:
    L: int
    H: int
    d: int
    ffn: int
    T: int
    C: int

    @property
    def dh(self) -> int:
        return self.d // self.H

    @property
    def fs(self) -> int:
        return self.ffn // self.H

    @property
    def K(self) -> int:
        return self.L * self.H


def unpack(cfg: Config, flat: np.ndarray) -> dict:
    """Views into the canonical flat vector (no copies)."""
    d, dh, fs, T, C, H = cfg.d, cfg.dh, cfg.fs, cfg.T, cfg.C, cfg.H
    off = 0

    def take(*shape):
        nonlocal off
        n = int(np.prod(shape))
        v = flat[off:off + n].reshape(shape)
        off += n
        return v

    p = {"w_embed": take(d, d), "b_embed": take(d), "pos": take(T, d), "blocks": []}
    for _ in range(cfg.K):
        p["blocks"].append({
            "wq": take(d, dh), "wk": take(d, dh), "wv": take(d, dh), "wo": take(dh, d),
            "w1": take(d, fs), "b1": take(fs), "w2": take(fs, d), "b2": take(d // H)})
    p["w_cls"] = take(d, C)
    p["b_cls"] = take(C)
    assert off == flat.size
    return p


def param_count(cfg: Config) -> int:
    d, dh, fs = cfg.d, cfg.dh, cfg.fs
    return d * d + d + cfg.T * d + cfg.K * (3 * d * dh + dh * d + d * fs + fs + fs * d + d // cfg.H) \
        + d * cfg.C + cfg.C


def subnet_slices(cfg: Config):
    """(start, stop) of each subnet (embed, K blocks, head) in the flat vector."""
    d, dh, fs = cfg.d, cfg.dh, cfg.fs
    e = d * d + d + cfg.T * d
    b = 3 * d * dh + dh * d + d * fs + fs + fs * d + d // cfg.H
    out = [(0, e)]
    for k in range(cfg.K):
        out.append((e + k * b, e + (k + 1) * b))
    out.append((e + cfg.K * b, e + cfg.K * b + d * cfg.C + cfg.C))
    return out


# linalg.cpp:133-151 (no affine)
def layer_norm(x):
    mean = x.mean(axis=1, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=1, keepdims=True)
    inv = 1.0 / np.sqrt(var + LN_EPS)
    return (x - mean) * inv


# linalg.cpp:153-180
def layer_norm_backward(x, dy):
    n = x.shape[1]
    mean = x.mean(axis=1, keepdims=True)
    var = ((x - mean) ** 2).mean(axis=1, keepdims=True)
    inv = 1.0 / np.sqrt(var + LN_EPS)
    y = (x - mean) * inv
    dy_mean = dy.sum(axis=1, keepdims=True) / n
    dy_dot = (dy * y).sum(axis=1, keepdims=True) / n
    return (dy - dy_mean - y * dy_dot) * inv


# linalg.cpp:182-188 (exact-erf GELU and its derivative)
def gelu(z):
    return 0.5 * z * (1.0 + _erf(z * 0.70710678118654752440))


def gelu_grad(z):
    return 0.5 * (1.0 + _erf(z * 0.70710678118654752440)) + z * 0.39894228040143267794 * np.exp(-0.5 * z * z)


def softmax_rows(s):
    m = s.max(axis=1, keepdims=True)
    e = np.exp(s - m)
    return e / e.sum(axis=1, keepdims=True)


def block_contribution(cfg, blk, h, xn, cache=None, ad=None, scaling=0.0):
    """model.cpp:197-241 (h is 0-based here; b2 offset = h*d/H, model.cpp:222).
    ad: LoRA adapters of the block subnet (model.cpp:204-211)."""
    q, k, v = xn @ blk["wq"], xn @ blk["wk"], xn @ blk["wv"]
    if ad is not None:
        pq, pk, pv = xn @ ad["down_q"], xn @ ad["down_k"], xn @ ad["down_v"]
        q = q + scaling * (pq @ ad["up_q"])
        k = k + scaling * (pk @ ad["up_k"])
        v = v + scaling * (pv @ ad["up_v"])
        if cache is not None:
            cache.update(pq=pq, pk=pk, pv=pv)
    probs = softmax_rows((q @ k.T) * (1.0 / math.sqrt(cfg.dh)))
    headout = probs @ v
    contrib = headout @ blk["wo"]
    z = xn @ blk["w1"] + blk["b1"]
    g = gelu(z)
    ffn = g @ blk["w2"]
    w = cfg.d // cfg.H
    ffn[:, h * w:(h + 1) * w] += blk["b2"]
    contrib = contrib + ffn
    if cache is not None:
        cache.update(xn=xn, q=q, k=k, v=v, probs=probs, headout=headout, z=z, g=g)
    return contrib


def contribution_backward(cfg, blk, h, c, dc, dxn, gb, ad=None, scaling=0.0, ga=None):
    """model.cpp:243-303; with adapters (ad, gradients into ga) the base
    tensors get no gradient (model.cpp:248-263, 273-289)."""
    lora = ad is not None
    dg = dc @ blk["w2"].T
    w = cfg.d // cfg.H
    if not lora:
        gb["w2"] += c["g"].T @ dc
        gb["b2"] += dc[:, h * w:(h + 1) * w].sum(axis=0)
    dz = dg * gelu_grad(c["z"])
    if not lora:
        gb["w1"] += c["xn"].T @ dz
        gb["b1"] += dz.sum(axis=0)
    dxn += dz @ blk["w1"].T
    dheadout = dc @ blk["wo"].T
    if not lora:
        gb["wo"] += c["headout"].T @ dc
    dprobs = dheadout @ c["v"].T
    dv = c["probs"].T @ dheadout
    dot = (c["probs"] * dprobs).sum(axis=1, keepdims=True)
    dscores = c["probs"] * (dprobs - dot)
    sc = 1.0 / math.sqrt(cfg.dh)
    dq = (dscores @ c["k"]) * sc
    dk = (dscores.T @ c["q"]) * sc
    for dproj, wname, x in ((dq, "wq", "q"), (dk, "wk", "k"), (dv, "wv", "v")):
        if lora:  # projection_backward, model.cpp:273-289
            ga["up_" + x] += scaling * (c["p" + x].T @ dproj)
            dp = scaling * (dproj @ ad["up_" + x].T)
            ga["down_" + x] += c["xn"].T @ dp
            dxn += dp @ ad["down_" + x].T
        else:
            gb[wname] += c["xn"].T @ dproj
        dxn += dproj @ blk[wname].T


def forward_backward(cfg: Config, flat: np.ndarray, inputs, labels, column, trace=None, lora=None, surrogate=None):
    """SubnetModel::forward_backward, model.cpp:416-520.

    Returns (loss, grads_flat, engaged[K+2]).  `trace`, if a dict, receives the
    block inputs per sample (for activation-level parity checks).
    lora = (rank, scaling, adapters_flat): adapters attached (model.cpp:165-195);
    then only the adapters get gradients and the result is
    (loss, adapter_grads_flat, engaged).
    surrogate = (rank, factors_flat): the opt-in p_s surrogate of the B200
    engine (d2ft_engine_set_surrogate; not a reference feature): a shortcut
    cell adds xn . down . up (per block subnet: down [d][R], up [R][d]),
    stop-gradient like p_o."""
    p = unpack(cfg, flat)
    sur = None
    if surrogate is not None:
        sr, sflat = surrogate
        per = 2 * cfg.d * sr
        sur = [(sflat[k * per:k * per + cfg.d * sr].reshape(cfg.d, sr),
                sflat[k * per + cfg.d * sr:(k + 1) * per].reshape(sr, cfg.d)) for k in range(cfg.K)]
    grads = np.zeros_like(flat)
    g = unpack(cfg, grads)
    ads = gads = None
    scaling = 0.0
    if lora is not None:
        rank, scaling, aflat = lora
        ads = lora_unpack(cfg, rank, aflat)
        agrads = np.zeros_like(aflat)
        gads = lora_unpack(cfg, rank, agrads)
    column = list(column)
    engaged = np.zeros(cfg.K + 2, dtype=np.uint8)
    engaged[0] = engaged[-1] = 1
    for r in range(cfg.K):
        if column[r] == 1:
            engaged[1 + r] = 1
    n = len(inputs)
    inv_n = 1.0 / n
    loss = 0.0
    L, H = cfg.L, cfg.H
    for si in range(n):
        inp = np.asarray(inputs[si], dtype=np.float64)
        x = inp @ p["w_embed"] + p["b_embed"] + p["pos"]
        xs = [x]
        caches = [None] * cfg.K
        for l in range(L):
            xin = xs[-1]
            xn = layer_norm(xin)
            acc = xin.copy()
            for h in range(H):
                r = l * H + h
                op = column[r]
                if op == 3:
                    if sur is not None:
                        acc += (xn @ sur[r][0]) @ sur[r][1]
                    continue
                cache = {} if op == 1 else None
                acc += block_contribution(cfg, p["blocks"][r], h, xn, cache, ads[r] if ads else None, scaling)
                caches[r] = cache
            xs.append(acc)
        if trace is not None:
            trace.setdefault("block_inputs", []).append([a.copy() for a in xs])
        fx = xs[-1]
        xn_h = layer_norm(fx)
        pooled = xn_h.mean(axis=0)
        logits = pooled @ p["w_cls"] + p["b_cls"]
        mx = logits.max()
        e = np.exp(logits - mx)
        ssum = e.sum()
        lab = int(labels[si])
        loss += (math.log(ssum) - (logits[lab] - mx)) * inv_n  # model.cpp:400-414
        dlogits = e / ssum
        dlogits[lab] -= 1.0
        dlogits *= inv_n
        if trace is not None:
            trace.setdefault("logits", []).append(logits.copy())
        g["w_cls"] += np.outer(pooled, dlogits)
        g["b_cls"] += dlogits
        dpooled = dlogits @ p["w_cls"].T
        dxn_h = np.broadcast_to(dpooled / cfg.T, fx.shape)
        dx = layer_norm_backward(fx, dxn_h)
        for l in range(L - 1, -1, -1):
            xin = xs[l]
            dxn = np.zeros_like(xin)
            anyf = False
            for h in range(H):
                r = l * H + h
                if column[r] != 1:
                    continue
                contribution_backward(cfg, p["blocks"][r], h, caches[r], dx, dxn, g["blocks"][r],
                                      ads[r] if ads else None, scaling, gads[r] if gads else None)
                anyf = True
            if anyf:
                dx = dx + layer_norm_backward(xin, dxn)
        g["w_embed"] += inp.T @ dx
        g["b_embed"] += dx.sum(axis=0)
        g["pos"] += dx
    if lora is not None:
        return loss, agrads, engaged
    return loss, grads, engaged


# ---------------------------------------------------------------- LoRA
def lora_block_size(cfg: Config, rank: int) -> int:
    return 3 * (cfg.d * rank + rank * cfg.dh)


def lora_unpack(cfg: Config, rank: int, aflat: np.ndarray):
    """Views per block subnet in visit_tensors order (model.hpp:139-146):
    down_q[d,r], up_q[r,dh], down_k, up_k, down_v, up_v."""
    d, dh = cfg.d, cfg.dh
    out, off = [], 0
    for _ in range(cfg.K):
        a = {}
        for x in "qkv":
            a["down_" + x] = aflat[off:off + d * rank].reshape(d, rank)
            off += d * rank
            a["up_" + x] = aflat[off:off + rank * dh].reshape(rank, dh)
            off += rank * dh
        out.append(a)
    assert off == aflat.size
    return out


def lora_init(cfg: Config, rank: int, seed: int) -> np.ndarray:
    """attach_lora (model.cpp:165-195): down = 0; up_q, up_k, up_v ~ N(0, 1/rank)
    from make_rng(seed, 0x10000 + subnet index), block subnet (l,h) at index
    1 + l*H + h (partition order, model.cpp:140-156)."""
    from oracle import lib as O
    aflat = np.zeros(cfg.K * lora_block_size(cfg, rank))
    ads = lora_unpack(cfg, rank, aflat)
    sd = 1.0 / math.sqrt(rank)
    for r in range(cfg.K):
        gs = O.gaussian_stream(seed, 0x10000 + 1 + r, 3 * rank * cfg.dh)
        for i, x in enumerate("qkv"):
            ads[r]["up_" + x][...] = (sd * gs[i * rank * cfg.dh:(i + 1) * rank * cfg.dh]).reshape(rank, cfg.dh)
    return aflat


def train_batch_lora(cfg: Config, flat, rank, scaling, aflat, avel, inputs, labels, codes, mbs, lr, momentum):
    """Trainer batch body with adapters attached (trainer.cpp:247-268,
    sgd_momentum_step over visit_trainable = adapters only, trainer.cpp:124-133);
    updates aflat / avel in place."""
    codes = np.asarray(codes, dtype=np.uint8).reshape(cfg.K, -1)
    n_mb = codes.shape[1]
    inv_mb = 1.0 / n_mb
    accum = np.zeros_like(aflat)
    touched = np.zeros(cfg.K, dtype=bool)
    batch_loss = 0.0
    for j in range(n_mb):
        loss, ga, eng = forward_backward(cfg, flat, inputs[j * mbs:(j + 1) * mbs], labels[j * mbs:(j + 1) * mbs],
                                         codes[:, j], lora=(rank, scaling, aflat))
        batch_loss += loss * inv_mb
        accum += ga * inv_mb
        touched |= eng[1:-1].astype(bool)
    bs = lora_block_size(cfg, rank)
    for r in range(cfg.K):
        if not touched[r]:
            continue
        a, b = r * bs, (r + 1) * bs
        avel[a:b] = momentum * avel[a:b] + accum[a:b]
        aflat[a:b] -= lr * avel[a:b]
    return batch_loss, touched


def train_batch(cfg: Config, flat: np.ndarray, velocity: np.ndarray, inputs, labels, codes, mbs,
                lr, momentum, surrogate=None):
    """Trainer batch body, trainer.cpp:247-268, updating flat/velocity in place.

    inputs: n_mb*mbs samples in unit order; codes: K x n_mb table."""
    codes = np.asarray(codes, dtype=np.uint8).reshape(cfg.K, -1)
    n_mb = codes.shape[1]
    inv_mb = 1.0 / n_mb
    accum = np.zeros_like(flat)
    touched = np.zeros(cfg.K + 2, dtype=bool)
    batch_loss = 0.0
    for j in range(n_mb):
        xs = inputs[j * mbs:(j + 1) * mbs]
        ls = labels[j * mbs:(j + 1) * mbs]
        loss, gr, eng = forward_backward(cfg, flat, xs, ls, codes[:, j], surrogate=surrogate)
        batch_loss += loss * inv_mb
        accum += gr * inv_mb
        touched |= eng.astype(bool)
    for si, (a, b) in enumerate(subnet_slices(cfg)):
        if not touched[si]:
            continue  # trainer.cpp:264-268: untouched subnets keep p and v
        g = accum[a:b]
        if not np.all(np.isfinite(g)):
            raise FloatingPointError("sgd: non-finite gradient")  # trainer.cpp:118
        velocity[a:b] = momentum * velocity[a:b] + g
        flat[a:b] -= lr * velocity[a:b]
    return batch_loss, touched


_PAR = {}


def _par_chunk(js):
    """Worker of train_batch_parallel: the micro-batches js in order, summed
    as the trainer does (accum += grads * (1/n_mb))."""
    from threadpoolctl import threadpool_limits
    a = _PAR
    with threadpool_limits(1):
        acc = np.zeros_like(a["flat"])
        losses, touched = [], np.zeros(a["cfg"].K + 2, dtype=bool)
        for j in js:
            mbs = a["mbs"]
            loss, gr, eng = forward_backward(a["cfg"], a["flat"], a["inputs"][j * mbs:(j + 1) * mbs],
                                             a["labels"][j * mbs:(j + 1) * mbs], a["codes"][:, j])
            acc += gr * a["inv_mb"]
            losses.append(loss)
            touched |= eng.astype(bool)
    return losses, acc, touched


def train_batch_parallel(cfg: Config, flat: np.ndarray, velocity: np.ndarray, inputs, labels, codes, mbs, lr,
                         momentum, workers=8):
    """train_batch with the micro-batches split over `workers` forked
    processes (test infrastructure for batch-64 ViT parity runs).  Each worker
    sums a contiguous run of micro-batches in order and the runs are summed in
    order, so the gradient differs from the serial trainer's left-to-right sum
    only by fp64 re-association (~1e-16 relative); the loss is summed in the
    serial order.  Updates flat / velocity in place like train_batch."""
    import multiprocessing as mp
    codes = np.asarray(codes, dtype=np.uint8).reshape(cfg.K, -1)
    n_mb = codes.shape[1]
    workers = max(1, min(workers, n_mb))
    _PAR.clear()
    _PAR.update(cfg=cfg, flat=flat, inputs=np.asarray(inputs, np.float64), labels=np.asarray(labels), codes=codes,
                mbs=mbs, inv_mb=1.0 / n_mb)
    bounds = np.linspace(0, n_mb, workers + 1).astype(int)
    runs = [list(range(bounds[i], bounds[i + 1])) for i in range(workers)]
    with mp.get_context("fork").Pool(workers) as pool:
        parts = pool.map(_par_chunk, runs)
    _PAR.clear()
    accum = np.zeros_like(flat)
    touched = np.zeros(cfg.K + 2, dtype=bool)
    batch_loss = 0.0
    for losses, acc, t in parts:
        for loss in losses:
            batch_loss += loss * (1.0 / n_mb)
        accum += acc
        touched |= t
    for si, (a, b) in enumerate(subnet_slices(cfg)):
        if not touched[si]:
            continue
        g = accum[a:b]
        if not np.all(np.isfinite(g)):
            raise FloatingPointError("sgd: non-finite gradient")
        velocity[a:b] = momentum * velocity[a:b] + g
        flat[a:b] -= lr * velocity[a:b]
    return batch_loss, touched


# scoring.cpp:57-96 (non-LoRA: every tensor of the block subnet) and
# prepass_scores, scoring.cpp:108-151: per unit, forward_backward with every
# scheduled subnet Full, then the metric of each head-subnet's unit gradient.
METRICS = ("fisher_information", "weight_magnitude", "gradient_magnitude", "taylor_importance")


def metric_value(metric, w, g):
    if metric == "fisher_information":
        return float(np.sum(g * g))
    if metric == "weight_magnitude":
        return float(np.sum(np.abs(w)))
    if metric == "gradient_magnitude":
        return float(np.sum(np.abs(g)))
    if metric == "taylor_importance":
        return float(np.sum(np.abs(w * g)))
    raise ValueError(metric)


def prepass_scores(cfg: Config, flat, inputs, labels, mbs, fwd_metric, bwd_metric):
    n = len(inputs)
    assert n % mbs == 0
    units = n // mbs
    sl = subnet_slices(cfg)
    fwd = np.zeros((cfg.K, units))
    bwd = np.zeros((cfg.K, units))
    col = np.ones(cfg.K, np.uint8)
    for u in range(units):
        _, g, _ = forward_backward(cfg, flat, inputs[u * mbs:(u + 1) * mbs], labels[u * mbs:(u + 1) * mbs], col)
        for k in range(cfg.K):
            a, b = sl[1 + k]
            fwd[k, u] = metric_value(fwd_metric, flat[a:b], g[a:b])
            bwd[k, u] = metric_value(bwd_metric, flat[a:b], g[a:b])
    return fwd, bwd


def prepass_scores_lora(cfg: Config, flat, rank, scaling, aflat, inputs, labels, mbs, fwd_metric, bwd_metric):
    """prepass_scores with adapters attached (scoring.cpp:129-148 with
    lora_enabled(): metric_value walks visit_trainable = the six adapter
    tensors of each block subnet, model.hpp:155-172)."""
    n = len(inputs)
    assert n % mbs == 0
    units = n // mbs
    bs = lora_block_size(cfg, rank)
    fwd = np.zeros((cfg.K, units))
    bwd = np.zeros((cfg.K, units))
    col = np.ones(cfg.K, np.uint8)
    for u in range(units):
        _, ga, _ = forward_backward(cfg, flat, inputs[u * mbs:(u + 1) * mbs], labels[u * mbs:(u + 1) * mbs], col,
                                    lora=(rank, scaling, aflat))
        for k in range(cfg.K):
            a, b = k * bs, (k + 1) * bs
            fwd[k, u] = metric_value(fwd_metric, aflat[a:b], ga[a:b])
            bwd[k, u] = metric_value(bwd_metric, aflat[a:b], ga[a:b])
    return fwd, bwd
