"""2-rank NCCL data parallelism on real GPUs (skipped on a 1-GPU box): the
batch-sharded greedy generation (parallel.dp_greedy_generate, reference loop
model.py:306-320 over independent sequences) equals the single-rank result bit
for bit, and bench.py --gpus 2 starts two NCCL ranks itself."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def _need2():
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, prompts, steps, q):
    import torch.distributed as dist

    sys.path.insert(0, str(ROOT / "tests"))
    from conftest import load_npz
    from fixtures_util import mirror_model

    from paper_2410_13229_b200.model import device_model
    from paper_2410_13229_b200.parallel import dp_greedy_generate

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    try:
        z, meta = load_npz("model_tiny2.npz")
        dm = device_model(mirror_model(z, meta))
        out = dp_greedy_generate(dm, prompts.cuda(), steps)
        q.put((rank, out.cpu().numpy()))
    finally:
        dist.destroy_process_group()


def test_dp_greedy_nccl_world2_bit_exact(cuda):
    _need2()
    from conftest import load_npz
    from fixtures_util import mirror_model

    from paper_2410_13229_b200.model import device_model

    rng = np.random.default_rng(4)
    prompts = torch.from_numpy(rng.integers(0, 256, size=(5, 12)))
    steps = 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, prompts, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    z, meta = load_npz("model_tiny2.npz")
    ref = device_model(mirror_model(z, meta)).greedy_generate(prompts.cuda(), steps).cpu().numpy()
    for rank, out in res:
        assert np.array_equal(out, ref), rank


def test_bench_spawns_two_nccl_ranks(cuda):
    _need2()
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "tiny", "--batch", "4",
                        "--seq", "64", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-extras"],
                       capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["comm"]["backend"] == "nccl" and line["comm"]["world_size"] == 2
