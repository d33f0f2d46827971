"""CPU: the product's host-side initialisation and synthetic data are
bit-identical to the (pinned) oracle — no GPU needed for these entry points."""
import numpy as np

from paper_2504_12471_b200 import engine as E
from oracle import lib as O


def test_partition_model_bit_identical():
    for cfg in (E.ModelConfig(2, 4, 32, 64, 16, 4, 1), E.ModelConfig(1, 2, 128, 256, 10, 3, 99), E.TINY):
        got = E.partition_model(cfg)
        ref = O.partition_model(cfg.num_blocks, cfg.heads_per_block, cfg.model_dim, cfg.ffn_hidden, cfg.seq_len,
                                cfg.num_classes, cfg.seed)
        assert np.array_equal(got, ref)


def test_synthetic_dataset_matches_fp32_rounding():
    x, y = E.make_synthetic_dataset(8, 4, 32, 16, 0.5, 7)
    rx, ry = O.make_dataset(8, 4, 32, 16, 0.5, 7)
    assert np.array_equal(x, rx.astype(np.float32)) and np.array_equal(y, ry)


def test_slices_cover_param_vector():
    cfg = E.TINY
    s = E.subnet_slices(cfg)
    assert s[0][0] == 0 and s[-1][1] == E.param_count(cfg) and len(s) == cfg.subnet_count()


def test_synthetic_dataset_f64_bit_identical_to_reference_dataset():
    """The fp64 Dataset (data.hpp) the step_units path ingests: every sample is
    the reference's Matrix bit for bit (golden data_x from the reference), each
    its own page-aligned allocation."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "rng_init.npz"))
    ds = E.make_synthetic_dataset_f64(8, 4, 32, 16, 0.5, 7)
    assert ds.size() == 8 and ds.num_classes == 4
    assert np.array_equal(np.stack(ds.samples), g["data_x"]) and np.array_equal(ds.labels, g["data_y"])
    assert all(s.ctypes.data % 4096 == 0 for s in ds.samples)
    assert ds.micro_batch_count(2) == 4
    assert np.array_equal(np.stack(ds.unit_inputs(1, 2)), g["data_x"][2:4])
    try:
        ds.micro_batch_count(3)
        raise AssertionError("expected input_error")
    except E.Error as e:
        assert e.kind == "input"
