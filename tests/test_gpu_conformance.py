"""Drop-in conformance on the GPU: build/conformance runs the reference's own
templates (hessian_matvec_with, pcg, Preconditioner<E>, objective) with
CudaEngine substituted for SerialEngine and compares with the serial run
(tests/conformance/conformance.cpp). Built by __graft_entry__.build() where
/root/reference is present; the binary travels to the GPU box."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "conformance")


@pytest.mark.skipif(not os.path.exists(EXE), reason="conformance binary not built (needs /root/reference)")
def test_reference_templates_on_cuda_engine():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    vals = dict(ln.split()[:2] for ln in r.stdout.splitlines() if len(ln.split()) == 2)
    for k in ("objective", "mismatch", "hessian_matvec", "pcg_5_inva", "precond_2linvh0"):
        assert float(vals[k]) <= 1e-4, (k, vals[k])
