"""Multi-process (gloo, world_size 2) tests of the batch-sharded DP host logic.
The per-rank model is the CPU oracle (a stand-in for the per-GPU DeviceModel),
so these run without a GPU; bit-exactness vs the single-process result is the
contract (sequences are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2410_13229_b200.parallel import shard_range


def test_shard_range_balanced_and_covering():
    for B in range(0, 40):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(B, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == B
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class _OracleDM:
    """Host stand-in with DeviceModel.greedy_generate's contract."""

    def __init__(self):
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parent))
        from conftest import load_npz
        from fixtures_util import oracle_model

        z, meta = load_npz("model_tiny2.npz")
        self.m = oracle_model(z, meta)

    def greedy_generate(self, prompts, steps):
        from oracle import oracle as o

        rows = [o.greedy(self.m, p.tolist(), steps) for p in prompts]
        return torch.tensor(rows, dtype=torch.int64)


def _worker(rank, world, port, prompts, steps, q):
    import torch.distributed as dist

    from paper_2410_13229_b200.parallel import dp_greedy_generate, gather_rows

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dm = _OracleDM()
        out = dp_greedy_generate(dm, prompts, steps)
        # ragged gather of float rows as well
        B = 5
        s, e = shard_range(B, rank, world)
        rows = torch.arange(s, e, dtype=torch.float32)[:, None].repeat(1, 3)
        full = gather_rows(rows, B)
        q.put((rank, out.numpy(), full.numpy()))
    finally:
        dist.destroy_process_group()


def test_dp_generate_world2_matches_single_process():
    rng = np.random.default_rng(4)
    prompts = torch.from_numpy(rng.integers(0, 256, size=(3, 6)))
    steps = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, prompts, steps, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = _OracleDM().greedy_generate(prompts, steps).numpy()
    for rank, out, full in res:
        assert np.array_equal(out, ref), rank
        assert np.array_equal(full[:, 0], np.arange(5, dtype=np.float32)), rank
