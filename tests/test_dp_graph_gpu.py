"""The N>1 bench step's CUDA graph (kernels + bucketed NCCL all-reduces captured
together, bench.py / model.GraphedStep with a reducer), exercised on the one GPU
this pool gives: a world-1 NCCL process group with the collectives forced on.
The captured step must replay bit-identically to the eager step."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_graph_captured_allreduce_step_matches_eager(cuda, prec):
    port = 29600 + (0 if prec == "fp32" else 1)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "workers", "dp_graph_worker.py"), prec],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert f"DP_GRAPH_OK {prec}" in r.stdout
