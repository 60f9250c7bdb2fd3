"""The library's NCCL path on one GPU: libnccl is dlopen'ed by the library itself
(context.cu), also inside a process where torch has already loaded its own NCCL (bench.py
under torchrun). stamg_nccl_selftest makes every NCCL call the sharded contexts make on a
one-rank communicator: unique id, ncclCommInitRank (the id passed by value), ncclCommSplit,
ncclAllReduce on a non-blocking stream, destroy; the sum over one rank must be the input."""
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SNIPPET = """
import sys
sys.path.insert(0, {root!r})
{pre}
from paper_2010_04559_b200 import stamg
v = stamg.nccl_selftest(0, 1 << 22)
print("nccl", v)
"""


@pytest.mark.parametrize("with_torch", [False, True])
def test_one_rank_round_trip(with_torch):
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pre = ("import torch, torch.distributed\ntorch.cuda.init()\n"
           "x = torch.ones(8, device='cuda')  # CUDA context + torch's libnccl mapped\n") if with_torch else ""
    r = subprocess.run([sys.executable, "-c", SNIPPET.format(root=root, pre=pre)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "nccl" in r.stdout and int(r.stdout.split()[-1]) >= 21800, r.stdout
