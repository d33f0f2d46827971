"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes bindings for
  * oracle/_build/liboracle.so — the plain-C restatement (sched_oracle.c), and
  * oracle/_ref/libd2ft_ref.so — the unmodified reference compiled from
    /root/reference by oracle/Makefile (absent on hosts where it was not built).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libd2ft_ref.so")

_P = C.c_void_p
_I = C.c_int
_U64 = C.c_uint64
_D = C.c_double


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def build(ref: bool = False) -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


_oracle = None
_ref = None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.or_param_count.restype = C.c_int64
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.ref_model_create.restype = C.c_void_p
        lib.ref_model_param_count.restype = C.c_uint64
        lib.ref_model_param_count.argtypes = [C.c_void_p]
        lib.ref_model_destroy.argtypes = [C.c_void_p]
        lib.ref_model_get_params.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_model_set_params.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_model_get_velocity.argtypes = [C.c_void_p, C.c_void_p]
        lib.ref_last_error.restype = C.c_char_p
        _ref = lib
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


# ------------------------------------------------------------------ C restatement
def uniform_stream(seed, stream, n):
    out = np.empty(n, np.float64)
    oracle_lib().or_uniform_stream(_U64(seed), _U64(stream), _I(n), _ptr(out))
    return out


def gaussian_stream(seed, stream, n):
    out = np.empty(n, np.float64)
    oracle_lib().or_gaussian_stream(_U64(seed), _U64(stream), _I(n), _ptr(out))
    return out


def shuffle_iota(seed, stream, n):
    out = np.empty(n, np.int32)
    oracle_lib().or_shuffle_iota(_U64(seed), _U64(stream), _I(n), _ptr(out))
    return out


def _rowcost(x, K):
    return np.ascontiguousarray(np.broadcast_to(np.asarray(x, np.int32), (K,)), np.int32)


def dp_search(scores, weights, caps):
    s = np.ascontiguousarray(scores, np.float64)
    K, N = s.shape
    w = np.ascontiguousarray(weights, np.int32)
    c = np.ascontiguousarray(caps, np.int32)
    sel = np.zeros((K, N), np.uint8)
    obj = np.zeros(K, np.float64)
    rc = oracle_lib().or_dp_search(_ptr(s), _ptr(w), _ptr(c), _I(K), _I(N), _ptr(sel), _ptr(obj))
    if rc:
        raise OracleError(rc)
    return sel, obj


def merge_selections(full_sel, fwd_sel):
    a = np.ascontiguousarray(full_sel, np.uint8)
    b = np.ascontiguousarray(fwd_sel, np.uint8)
    K, N = a.shape
    codes = np.zeros((K, N), np.uint8)
    oracle_lib().or_merge_selections(_ptr(a), _ptr(b), _I(K), _I(N), _ptr(codes))
    return codes


def knapsack_schedule(bwd, fwd, cf, cb, cap_full, cap_fwd):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    rc = oracle_lib().or_knapsack_schedule(
        _ptr(b), _ptr(f), _ptr(_rowcost(cf, K)), _ptr(_rowcost(cb, K)),
        _ptr(np.ascontiguousarray(cap_full, np.int32)), _ptr(np.ascontiguousarray(cap_fwd, np.int32)),
        _I(K), _I(N), _ptr(codes))
    if rc:
        raise OracleError(rc)
    return codes


def scaler_schedule(bwd, fwd, cf, cb, total_cap, mode, lam=1.0):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    lu = C.c_double()
    fb = C.c_int()
    rc = oracle_lib().or_scaler_schedule(
        _ptr(b), _ptr(f), _ptr(_rowcost(cf, K)), _ptr(_rowcost(cb, K)),
        _ptr(np.ascontiguousarray(total_cap, np.int32)), _I(K), _I(N), _I(mode), _D(lam), _ptr(codes),
        C.byref(lu), C.byref(fb))
    if rc:
        raise OracleError(rc)
    return codes, lu.value, bool(fb.value)


def brute_force_schedule(bwd, fwd, cf, cb, cap_full, cap_fwd):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    rc = oracle_lib().or_brute_force_schedule(
        _ptr(b), _ptr(f), _ptr(_rowcost(cf, K)), _ptr(_rowcost(cb, K)),
        _ptr(np.ascontiguousarray(cap_full, np.int32)), _ptr(np.ascontiguousarray(cap_fwd, np.int32)),
        _I(K), _I(N), _ptr(codes))
    if rc:
        raise OracleError(rc)
    return codes


def compact(codes, H):
    c = np.ascontiguousarray(codes, np.uint8)
    K, N = c.shape
    L = K // H
    fwd_idx = np.full((K, N), -1, np.int32)
    full_idx = np.full((K, N), -1, np.int32)
    fwd_cnt = np.zeros(K, np.int32)
    full_cnt = np.zeros(K, np.int32)
    act = np.full((N * L, H), -1, np.int32)
    fullh = np.full((N * L, H), -1, np.int32)
    act_cnt = np.zeros(N * L, np.int32)
    full_hcnt = np.zeros(N * L, np.int32)
    oracle_lib().or_compact(_ptr(c), _I(K), _I(N), _I(H), _ptr(fwd_idx), _ptr(fwd_cnt), _ptr(full_idx),
                            _ptr(full_cnt), _ptr(act), _ptr(act_cnt), _ptr(fullh), _ptr(full_hcnt))
    return dict(fwd_idx=fwd_idx, fwd_cnt=fwd_cnt, full_idx=full_idx, full_cnt=full_cnt,
                act_heads=act, act_cnt=act_cnt, full_heads=fullh, full_hcnt=full_hcnt)


def partition_model(L, H, d, ffn, T, C_, seed):
    n = oracle_lib().or_param_count(_I(L), _I(H), _I(d), _I(ffn), _I(T), _I(C_))
    out = np.empty(n, np.float64)
    oracle_lib().or_partition_model(_I(L), _I(H), _I(d), _I(ffn), _I(T), _I(C_), _U64(seed), _ptr(out))
    return out


def make_dataset(num_samples, C_, d, T, noise, seed):
    samples = np.empty((num_samples, T, d), np.float64)
    labels = np.empty(num_samples, np.int32)
    rc = oracle_lib().or_make_dataset(_I(num_samples), _I(C_), _I(d), _I(T), _D(noise), _U64(seed),
                                      _ptr(samples), _ptr(labels))
    if rc:
        raise OracleError(rc)
    return samples, labels


def random_score_table(K, N, seed, zero_prob=0.0):
    """test_scheduler.cpp:15-34 (random_score_table): f then b per cell, row-major,
    with the optional zeroing draws, all from make_rng(seed, 0)."""
    per = 4 if zero_prob > 0.0 else 2
    u = uniform_stream(seed, 0, K * N * per)
    f = np.empty((K, N))
    b = np.empty((K, N))
    it = 0
    for k in range(K):
        for j in range(N):
            fv = u[it] * 10.0
            bv = u[it + 1] * 10.0
            it += 2
            if zero_prob > 0.0:
                if u[it] < zero_prob:
                    fv = 0.0
                it += 1
                if u[it] < zero_prob:
                    bv = 0.0
                it += 1
            f[k, j] = fv
            b[k, j] = bv
    return b, f


def bench_scores(K, N, seed=1):
    """bench_scheduler.cpp:13-27 (make_scores): forward then backward per cell."""
    u = uniform_stream(seed, 0, 2 * K * N).reshape(K, N, 2)
    return u[:, :, 1] * 10.0, u[:, :, 0] * 10.0   # (bwd, fwd)


# ------------------------------------------------------------------ reference (oracle/_ref)
class RefModel:
    """The unmodified reference SubnetModel + its trainer body (ref_shim.cpp)."""

    def __init__(self, L, H, d, ffn, T, C_, seed):
        self.lib = ref_lib()
        self.h = self.lib.ref_model_create(_I(L), _I(H), _I(d), _I(ffn), _I(T), _I(C_), _U64(seed))
        if not self.h:
            raise OracleError(-1, self.lib.ref_last_error().decode())
        self.dims = (L, H, d, ffn, T, C_)
        self.n = int(self.lib.ref_model_param_count(self.h))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.ref_model_destroy(self.h)
            self.h = None

    def params(self):
        out = np.empty(self.n, np.float64)
        self.lib.ref_model_get_params(self.h, _ptr(out))
        return out

    def set_params(self, flat):
        a = np.ascontiguousarray(flat, np.float64)
        self.lib.ref_model_set_params(self.h, _ptr(a))

    def attach_lora(self, rank, scaling):
        rc = self.lib.ref_model_attach_lora(C.c_void_p(self.h), _I(rank), _D(scaling))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        self.lib.ref_model_flat_count.restype = C.c_int64
        self.n = int(self.lib.ref_model_flat_count(C.c_void_p(self.h)))

    def velocity(self):
        out = np.empty(self.n, np.float64)
        self.lib.ref_model_get_velocity(self.h, _ptr(out))
        return out

    def forward_backward(self, inputs, labels, column):
        x = np.ascontiguousarray(inputs, np.float64)
        lab = np.ascontiguousarray(labels, np.int32)
        col = np.ascontiguousarray(column, np.uint8)
        loss = C.c_double()
        grads = np.empty(self.n, np.float64)
        eng = np.zeros(self.dims[0] * self.dims[1] + 2, np.uint8)
        rc = self.lib.ref_forward_backward(C.c_void_p(self.h), _ptr(x), _ptr(lab), _I(len(lab)), _ptr(col),
                                           C.byref(loss), _ptr(grads), _ptr(eng))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return loss.value, grads, eng

    def prepass_scores(self, inputs, labels, mbs, fwd_metric, bwd_metric, threads=1):
        """The reference's prepass_scores (scoring.cpp:108-151); metrics as Metric enum ints."""
        x = np.ascontiguousarray(inputs, np.float64)
        lab = np.ascontiguousarray(labels, np.int32)
        units = len(lab) // mbs
        K = self.dims[0] * self.dims[1]
        fo = np.empty((K, units), np.float64)
        bo = np.empty((K, units), np.float64)
        rc = self.lib.ref_prepass_scores(C.c_void_p(self.h), _ptr(x), _ptr(lab), _I(len(lab)), _I(mbs),
                                         _I(fwd_metric), _I(bwd_metric), _I(threads), _ptr(fo), _ptr(bo))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return fo, bo

    def train_batch_parallel(self, inputs, labels, codes, mbs, lr, momentum, threads):
        x = np.ascontiguousarray(inputs, np.float64)
        lab = np.ascontiguousarray(labels, np.int32)
        c = np.ascontiguousarray(codes, np.uint8)
        loss = C.c_double()
        rc = self.lib.ref_train_batch_parallel(C.c_void_p(self.h), _ptr(x), _ptr(lab), _I(c.shape[1]), _I(mbs),
                                               _ptr(c), _D(lr), _D(momentum), _I(threads), C.byref(loss))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return loss.value

    def train_batch(self, inputs, labels, codes, mbs, lr, momentum):
        x = np.ascontiguousarray(inputs, np.float64)
        lab = np.ascontiguousarray(labels, np.int32)
        c = np.ascontiguousarray(codes, np.uint8)
        n_mb = c.shape[1]
        loss = C.c_double()
        rc = self.lib.ref_train_batch(C.c_void_p(self.h), _ptr(x), _ptr(lab), _I(n_mb), _I(mbs), _ptr(c),
                                      _D(lr), _D(momentum), C.byref(loss))
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())
        return loss.value


def ref_dp_search(scores, weights, caps, threads=1):
    s = np.ascontiguousarray(scores, np.float64)
    K, N = s.shape
    w = np.ascontiguousarray(weights, np.int32)
    c = np.ascontiguousarray(caps, np.int32)
    sel = np.zeros((K, N), np.uint8)
    obj = np.zeros(K, np.float64)
    rc = ref_lib().ref_dp_search(_ptr(s), _ptr(w), _ptr(c), _I(K), _I(N), _I(threads), _ptr(sel), _ptr(obj))
    if rc:
        raise OracleError(rc, ref_lib().ref_last_error().decode())
    return sel, obj


def ref_knapsack_schedule(bwd, fwd, cf, cb, cap_full, cap_fwd, threads=1, cf_dev=None, cb_dev=None):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    cfd = None if cf_dev is None else np.ascontiguousarray(cf_dev, np.int32)
    cbd = None if cb_dev is None else np.ascontiguousarray(cb_dev, np.int32)
    rc = ref_lib().ref_knapsack_schedule(
        _ptr(b), _ptr(f), _I(cf), _I(cb), None if cfd is None else _ptr(cfd), None if cbd is None else _ptr(cbd),
        _ptr(np.ascontiguousarray(cap_full, np.int32)), _ptr(np.ascontiguousarray(cap_fwd, np.int32)),
        _I(K), _I(N), _I(threads), _ptr(codes))
    if rc:
        raise OracleError(rc, ref_lib().ref_last_error().decode())
    return codes


def ref_scaler_schedule(bwd, fwd, cf, cb, total_cap, mode, lam=1.0, threads=1):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    lu = C.c_double()
    fb = C.c_int()
    rc = ref_lib().ref_scaler_schedule(_ptr(b), _ptr(f), _I(cf), _I(cb),
                                       _ptr(np.ascontiguousarray(total_cap, np.int32)), _I(K), _I(N), _I(mode),
                                       _D(lam), _I(threads), _ptr(codes), C.byref(lu), C.byref(fb))
    if rc:
        raise OracleError(rc, ref_lib().ref_last_error().decode())
    return codes, lu.value, bool(fb.value)


def ref_brute_force_schedule(bwd, fwd, cf, cb, cap_full, cap_fwd):
    b = np.ascontiguousarray(bwd, np.float64)
    f = np.ascontiguousarray(fwd, np.float64)
    K, N = b.shape
    codes = np.zeros((K, N), np.uint8)
    rc = ref_lib().ref_brute_force_schedule(_ptr(b), _ptr(f), _I(cf), _I(cb),
                                            _ptr(np.ascontiguousarray(cap_full, np.int32)),
                                            _ptr(np.ascontiguousarray(cap_fwd, np.int32)), _I(K), _I(N),
                                            _ptr(codes))
    if rc:
        raise OracleError(rc, ref_lib().ref_last_error().decode())
    return codes


def ref_make_dataset(num_samples, C_, d, T, noise, seed):
    samples = np.empty((num_samples, T, d), np.float64)
    labels = np.empty(num_samples, np.int32)
    rc = ref_lib().ref_make_dataset(_I(num_samples), _I(C_), _I(d), _I(T), _D(noise), _U64(seed),
                                    _ptr(samples), _ptr(labels))
    if rc:
        raise OracleError(rc, ref_lib().ref_last_error().decode())
    return samples, labels


def ref_uniform_stream(seed, stream, n):
    out = np.empty(n, np.float64)
    ref_lib().ref_uniform_stream(_U64(seed), _U64(stream), _I(n), _ptr(out))
    return out


def ref_shuffle_iota(seed, stream, n):
    out = np.empty(n, np.int32)
    ref_lib().ref_shuffle_iota(_U64(seed), _U64(stream), _I(n), _ptr(out))
    return out


# ------------------------------------------------------------------ reference artifact formats
# (oracle/ref_serialize_shim.cpp over the unmodified serialize.cpp)
def _ref_text(fn, *args):
    cap = 1 << 16
    while True:
        buf = C.create_string_buffer(cap)
        n = C.c_size_t()
        rc = fn(*args, buf, C.c_size_t(cap), C.byref(n))
        if rc == 6 and n.value + 1 > cap:
            cap = n.value + 1
            continue
        if rc:
            ref_lib().ref_ser_last_error.restype = C.c_char_p
            raise OracleError(rc, ref_lib().ref_ser_last_error().decode())
        return buf.raw[:n.value].decode()


def ref_format_double(v):
    return _ref_text(ref_lib().ref_ser_format_double, _D(v))


def ref_score_table_text(fwd, bwd, fwd_metric, bwd_metric, fmt):
    f = np.ascontiguousarray(fwd, np.float64)
    b = np.ascontiguousarray(bwd, np.float64).reshape(f.shape)
    K, N = f.shape
    if f.size == 0:
        f = b = np.zeros(1)
    return _ref_text(ref_lib().ref_ser_score_table, _I(K), _I(N), _ptr(f), _ptr(b), _I(fwd_metric), _I(bwd_metric),
                     _I(fmt))


def ref_schedule_table_text(codes, fmt):
    c = np.ascontiguousarray(codes, np.uint8)
    K, N = c.shape
    return _ref_text(ref_lib().ref_ser_schedule_table, _I(K), _I(N), _ptr(c), _I(fmt))


def ref_batch_metrics_text(m5, busy, run_id, method, fmt):
    m = np.ascontiguousarray(m5, np.float64)
    b = np.ascontiguousarray(busy if len(busy) else [0.0], np.float64)
    return _ref_text(ref_lib().ref_ser_batch_metrics, _ptr(m), _ptr(b), _I(len(busy)), run_id.encode(),
                     method.encode(), _I(fmt))


def ref_history_text(epochs, fmt):
    n = len(epochs)
    cols = [np.ascontiguousarray([e[i] for e in epochs] or [0], np.int32 if i == 0 else np.float64) for i in range(5)]
    return _ref_text(ref_lib().ref_ser_history, _I(n), *[_ptr(c) for c in cols], _I(fmt))


def ref_reparse(kind, text):
    """kind: 'score' / 'schedule' (re-emitted as JSON) or 'history' (as CSV)."""
    fn = {"score": ref_lib().ref_ser_score_table_reparse, "schedule": ref_lib().ref_ser_schedule_table_reparse,
          "history": ref_lib().ref_ser_history_reparse}[kind]
    return _ref_text(fn, text.encode())
