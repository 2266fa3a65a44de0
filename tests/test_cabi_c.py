"""The compiled C client of include/cpfit_gpu.h (tests/c/test_cabi.c, built by
__graft_entry__.build()): it includes the header from plain C11, links libcpfit_gpu.so and calls
cpfit_tensor_create_dense / cpfit_mttkrp / cpfit_objective_and_gradient / cpfit_ngmres_solve /
cpfit_tensor_create_coo against the reference's known answers."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "c", "_build", "test_cabi")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "c")], check=True)
    assert os.path.exists(BIN)


def test_c_client_builds_and_fails_loudly_without_gpu(P):
    _build()
    if P.device_count() > 0:
        pytest.skip("a GPU is visible (the gpu-marked test runs the client)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "fail loudly" in r.stdout


@pytest.mark.gpu
def test_c_client_on_gpu(gpu):
    _build()
    r = subprocess.run([BIN, "--expect-gpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "all C-ABI checks passed" in r.stdout
