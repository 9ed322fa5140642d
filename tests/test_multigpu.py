"""Real-NCCL multi-GPU parity: world 2 / 4 / 8 Morton-range
shards, one process per GPU, on BASELINE configs 1 and 3.  The job totals must
equal the single-GPU engine's to 1e-12 and the reference's goldens to 1e-10.
Runs whenever at least two GPUs are visible (skips only on a one-GPU box)."""
import json
import os
import socket
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _golden(config):
    name = {1: ("golden_big.json", "c1_L4"), 3: ("golden_c3.json", None)}[config]
    with open(os.path.join(HERE, "golden", name[0])) as f:
        d = json.load(f)
    if name[1] is None:
        return d["system"]["energies"]
    return next(s for s in d["systems"] if s["name"] == name[1])["energies"]


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
def test_nccl_shards_match_single_gpu_and_reference(cuda, world, tmp_path):
    torch = cuda
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU)")
    if world > ngpu:
        pytest.skip(f"world {world} > {ngpu} visible GPUs")
    import paper_2212_08284_b200 as ankh
    from paper_2212_08284_b200 import inputs

    out = tmp_path / "mgpu.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(HERE, "mgpu_worker.py"), str(out), "1", "3"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    got = json.loads(out.read_text())
    assert got["world"] == world
    for c in (1, 3):
        pos, src, rb, cfg = inputs.make_config(c)
        L = cfg.orders[0]
        single = ankh.Plan(pos.shape[0], rb, ankh.EwaldConfig(order_cheb=L, order_equi=L))
        s = single.energy(pos, src)
        single.close()
        res = got["results"][str(c)]
        assert res["pairs_total"] == s.near_pairs
        want = [s.e_total, s.e_self, s.e_near, s.e_far, s.e_periodic_far]
        for vals in res["device"] + [res["host"]]:
            for g, w in zip(vals, want):
                assert abs(g - w) <= 1e-12 * abs(want[0]), (c, vals, want)
        gold = float(_golden(c)["e_total"])
        assert abs(res["host"][0] - gold) <= 1e-10 * abs(gold)
