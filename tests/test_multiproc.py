"""N > 1 plumbing on CPU (gloo, world size 2): bench.py runs one independent
replica per rank (no data-path collective) and reports the
max over ranks of the device-timed region.  Also the reference arm's JSON
contract (the oracle timed on host cores)."""
import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        got = bench.max_over_ranks(10.0 + 5.0 * rank, ws)
        out.put((rank, got))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_max_over_ranks_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: 15.0, 1: 15.0}


def test_kernel_bytes_formula():
    sys.path.insert(0, ROOT)
    import bench
    # c5: 4,194,304 elements, 4,276,737 nodes, 12,830,211 DOFs
    kb = bench.kernel_bytes(3, 4194304, 4276737, 12830211, True)
    assert kb["k1"] == 8 * 4194304 + 8 * 4276737 + 64 * 12830211
    assert abs(kb["k1"] / 1e6 - 888.9) < 0.1
    assert kb["k2"] == 0
    # the deferred x update: 249 of 500 launches read and write x (kernels 2, 4, ..., 498)
    assert bench.x_touch_fraction(500) == 249 / 500 and bench.x_touch_fraction(1) == 0.0
    kb = bench.kernel_bytes(3, 4194304, 4276737, 12830211, True, 500)
    assert kb["k1"] == 8 * 4194304 + 8 * 4276737 + 48 * 12830211 + round(16 * 12830211 * 249 / 500)
    assert abs(kb["k1"] / 1e6 - 785.85) < 0.01


def test_reference_arm_json_contract():
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0",
                        "--ref-budget", "0.5"], cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "iterations/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0
