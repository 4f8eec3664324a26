"""Drop-in check at the reference's own API: build/integration_test runs the
reference's PolicyWorker and Cluster (compiled from /root/reference into
oracle/_ref) next to the B200 worker adapter (integration/) and compares
their replies (tests/cpp/integration_main.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "integration_test")
REF = "/root/reference/proj/core/include"


def test_integration_binary_builds_against_reference_headers():
    if not os.path.isdir(REF):
        pytest.skip("reference headers absent (GPU box): the binary is built in the CPU container")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    assert os.path.exists(BIN)


@pytest.mark.gpu
def test_reference_workers_vs_b200_worker():
    if not os.path.exists(BIN):
        pytest.skip("build/integration_test not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK (0 failures)")


TRAINER = os.path.join(ROOT, "build", "trainer_step")


def test_cpp_trainer_example_builds():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    assert os.path.exists(TRAINER)


@pytest.mark.gpu
def test_cpp_trainer_example_runs():
    """A C++ trainer through include/rlo.hpp only: GRPO step over micro-batches,
    the fused loss + dlogits pass (same loss), decode (examples/trainer_step.cpp)."""
    if not os.path.exists(TRAINER):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    r = subprocess.run([TRAINER], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")
