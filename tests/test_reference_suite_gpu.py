"""GPU: the reference's OWN scheduler test suite (proj/tests/test_scheduler.cpp,
unmodified) linked against the B200 binding (integration/d2ft_b200_binding.cpp
over libd2ft_b200.so) in place of core/src/scheduler.cpp.  The binary is built
here by `make -C oracle ref-tests` (needs /root/reference) and travels to the
GPU box in oracle/_ref/."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B200 = os.path.join(ROOT, "oracle", "_ref", "test_scheduler_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "test_scheduler_ref")


@pytest.mark.gpu
def test_reference_scheduler_suite_on_b200():
    if not os.path.exists(B200):
        pytest.skip("oracle/_ref/test_scheduler_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([B200], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout


def test_reference_scheduler_suite_on_reference_cpu():
    """Sanity of the doctest shim: the same suite passes on the reference itself."""
    if not os.path.exists(REF):
        pytest.skip("oracle/_ref/test_scheduler_ref not built")
    r = subprocess.run([REF], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "failed: 0" in r.stdout, r.stdout[-3000:]


TRAINER = os.path.join(ROOT, "oracle", "_ref", "test_b200_model_trainer")


@pytest.mark.gpu
def test_reference_operator_and_trainer_cases_on_b200():
    """The reference's test_model.cpp / test_trainer.cpp cases (adapted to the
    B200 tile sizes, integration/tests/test_b200_model_trainer.cpp) through the
    operator / trainer binding (integration/d2ft_b200_trainer.cpp): device
    forward_backward, logits / evaluate, the train() loop for every policy,
    update locality, cost fractions, LoRA freezing, failure before mutation."""
    if not os.path.exists(TRAINER):
        pytest.skip("oracle/_ref/test_b200_model_trainer not built (needs /root/reference at build time)")
    r = subprocess.run([TRAINER], capture_output=True, text=True, timeout=900)
    print(r.stdout[-3000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "failed: 0" in r.stdout
