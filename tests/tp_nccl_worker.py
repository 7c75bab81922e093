"""Rank body of test_tp_model_graph_nccl: one NCCL rank on the single GPU, the TP model
(DistComm) decode step captured as a CUDA graph with its collectives, replays
bit-identical to DeviceModel's eager decode."""
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))
sys.path.insert(0, str(HERE.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda:0"))
    rank, world = dist.get_rank(), dist.get_world_size()
    from conftest import load_npz
    from fixtures_util import mirror_model

    from paper_2410_13229_b200.model import device_model
    from paper_2410_13229_b200.tp import DistComm, TPModel

    z, meta = load_npz("model_config1.npz")
    qm = mirror_model(z, meta)
    dm = device_model(qm)
    tp = TPModel(qm, DistComm(), [rank], world)
    tok = torch.from_numpy(z["tokens"][None, :32].astype(np.int64)).cuda().repeat(2, 1)
    s_ref = dm.new_states(2)
    dm.prefill(tok, s_ref)
    s_tp = tp.new_states(2)
    tp.prefill(tok, s_tp)
    graph, tin, tout = tp.capture_decode(s_tp)
    cur = tok[:, -1].contiguous()
    for step in range(4):
        want = dm.decode_step(cur, s_ref)
        tin.copy_(cur)
        graph.replay()
        torch.cuda.synchronize()
        assert np.array_equal(tout.cpu().numpy().view(np.uint32), want.cpu().numpy().view(np.uint32)), step
        cur = want.argmax(-1)
    print("tp graph rank ok", rank, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
