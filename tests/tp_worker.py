"""Rank body of test_tp_block_two_processes_gloo (launched by torch.distributed.run)."""
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from fixtures_util import block_weights, load_block, mirror_block  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    from paper_2410_13229_b200.qblock import device_block
    from paper_2410_13229_b200.tp import DistComm, TPBlock, tp_block_forward

    z, meta = load_block("s2p8b")
    qb = mirror_block(z, meta, block_weights(z, meta))
    D = meta["cfg"]["d_model"]
    B, T = 2, 5
    rng = np.random.default_rng(5)
    u = torch.from_numpy(rng.integers(-127, 128, size=(B * T, D)).astype(np.int8)).cuda()
    want = torch.empty((B * T, D), dtype=torch.float32, device="cuda")
    device_block(qb).prefill(u, B, T, want, u_scale=meta["u_scale"])
    shard = TPBlock(qb, rank, world)
    got = torch.empty_like(want)
    tp_block_forward([shard], DistComm(), u, B, T, [got], u_scale=meta["u_scale"])
    torch.cuda.synchronize()
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want.cpu().numpy().view(np.uint32))
    print("tp rank ok", rank, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
