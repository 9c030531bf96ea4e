"""The tensor engine's alternative schedules stay bit-exact: the dynamic stream-K
claims with the end-of-work barrier (PB_TC_STATIC=0) and the static split with a
dynamic tail (PB_TC_DYN), each in a fresh process (the knobs are read once), on
shapes with many units per CTA, shared tiles, two accumulator groups and batch slices."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2003_00822_b200 as pb, synth, oracle
for (R, K, B, L, k, a) in [(4096, 8192, 1, 8, 8, 16), (4000, 8192, 1, 16, 11, 16), (1029, 784, 1, 4, 4, 16),
                           (300, 2000, 4, 8, 8, 16), (200, 1500, 37, 4, 4, 16)]:
    s = synth.seed(9, R + K + B)
    m = synth.codes(R, K, L, s)
    x = synth.inject_edges(synth.activations(B, K, s + 1, "gauss"), s + 2)
    w = pb.PackedWeights.from_codes(m, L, 0, 0.5)
    ws = pb.Workspace(pb.workspace_bytes(B, K, a))
    acc_o, y_o, _ = oracle.pbatch(m, L, 0, 0.5, k, x, a, nthreads=8)
    for rep in range(2):
        acc = torch.zeros((B, R), dtype=torch.int64, device="cuda")
        y = pb.matmul(torch.from_numpy(x).cuda(), w, k, a, acc=acc, ws=ws)
        torch.cuda.synchronize()
        assert np.array_equal(acc.cpu().numpy(), acc_o), (R, K, B, L, rep)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), y_o.view(np.uint32)), (R, K, B, L, rep)
print("ok")
'''


@pytest.mark.parametrize("env", [{"PB_TC_STATIC": "0"}, {"PB_TC_DYN": "10"}, {"PB_TC_DYN": "50"}])
def test_schedule_knobs_bit_exact(env):
    import build_pb
    build_pb.build()
    e = dict(os.environ)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + CHILD], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-2000:]
