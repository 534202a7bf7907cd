"""The distributed step on a real NCCL communicator (one rank on cuda:0, in its own process):
partition, window all_gather, halo plan, overlapped split step and the max-over-ranks
all_reduce — bitwise the single-GPU step.  (This run has one GPU: the multi-rank exchange itself
is covered by the gloo tests and the one-GPU emulations.)"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["cfg4", "cfg3", "cfg2"])
def test_nccl_one_rank_split_step(name):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    res = subprocess.run([sys.executable, os.path.join(HERE, "nccl_one_rank.py"), name, str(_free_port())],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    out = json.loads(res.stdout.strip().splitlines()[-1])
    assert out["backend"] == "nccl" and out["world"] == 1 and out["bitwise"]
