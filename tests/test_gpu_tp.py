"""Tensor-parallel E-sharding: G channel shards with int32
all-reduces of the x_proj / out_proj partial products and a gathered Hadamard
input reproduce the unsharded block bit for bit -- prefill (with exported
states) and carried-state decode."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from fixtures_util import block_weights, load_block, mirror_block

pytestmark = pytest.mark.gpu


def _bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("name,G", [("m20_full", 2), ("p2_naive", 2), ("p2_naive", 4), ("m12_full", 2),
                                    ("s130m", 2), ("s130m", 4), ("s2p8b", 2), ("s2p8b", 8)])
def test_tp_block_bit_exact(cuda, name, G):
    from paper_2410_13229_b200.qblock import device_block
    from paper_2410_13229_b200.tp import TPBlock, VirtualComm, tp_block_forward

    z, meta = load_block(name)
    qb = mirror_block(z, meta, block_weights(z, meta))
    ref = device_block(qb)
    D, E = meta["cfg"]["d_model"], meta["cfg"]["d_inner"]
    B, T = 3, 9
    rng = np.random.default_rng(G * 100 + E)
    u = torch.from_numpy(rng.integers(-127, 128, size=(B * T, D)).astype(np.int8)).cuda()
    out = torch.empty((B * T, D), dtype=torch.float32, device="cuda")
    conv, h = ref.new_state(B)
    ref.prefill(u, B, T, out, u_scale=meta["u_scale"], conv_state_out=conv, ssm_state_out=h)
    shards = [TPBlock(qb, r, G) for r in range(G)]
    comm = VirtualComm(G)
    outs = [torch.empty_like(out) for _ in range(G)]
    states = [s.new_state(B) for s in shards]
    tp_block_forward(shards, comm, u, B, T, outs, states=states, u_scale=meta["u_scale"])
    for r in range(G):
        assert np.array_equal(_bits(outs[r]), _bits(out)), r
        El = E // G
        assert np.array_equal(states[r][0].cpu().numpy(), conv[:, :, r * El:(r + 1) * El].cpu().numpy())
        assert np.array_equal(_bits(states[r][1]), _bits(h[:, r * El:(r + 1) * El]))
    # two decode steps from the exported states, accumulated into a residual
    for step in range(2):
        ud = torch.from_numpy(rng.integers(-127, 128, size=(B, D)).astype(np.int8)).cuda()
        res = torch.from_numpy(rng.standard_normal((B, D)).astype(np.float32)).cuda()
        want = res.clone()
        ref.decode(ud, conv, h, want, u_scale=meta["u_scale"], accumulate=True)
        got = [res.clone() for _ in range(G)]
        tp_block_forward(shards, comm, ud, B, 1, got, decode=True, states=states, accumulate=True,
                         u_scale=meta["u_scale"])
        for r in range(G):
            assert np.array_equal(_bits(got[r]), _bits(want)), (step, r)


def test_tp_block_two_processes_gloo(cuda):
    """The same decomposition with real torch.distributed collectives: two ranks
    (gloo, both on cuda:0 -- the single-GPU box), outputs bit-identical to the
    unsharded block."""
    here = Path(__file__).resolve().parent
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29500 + os.getpid() % 1000))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", env["MASTER_PORT"],
                        str(here / "tp_worker.py")], env=env, capture_output=True, text=True, timeout=600,
                       cwd=str(here.parent))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("tp rank ok") == 2, r.stdout[-2000:]


@pytest.mark.parametrize("G", [2, 4])
def test_tp_model_bit_exact(cuda, G):
    """The whole model loop over TP blocks (config1: d_model 256, 4 layers):
    hidden states of a prefill and the logits of carried-state decode steps equal
    DeviceModel's bit for bit."""
    from conftest import load_npz
    from fixtures_util import mirror_model

    from paper_2410_13229_b200.model import device_model
    from paper_2410_13229_b200.tp import TPModel, VirtualComm

    z, meta = load_npz("model_config1.npz")
    qm = mirror_model(z, meta)
    dm = device_model(qm)
    tp = TPModel(qm, VirtualComm(G), list(range(G)), G)
    tok = torch.from_numpy(z["tokens"][None, :64].astype(np.int64)).cuda().repeat(2, 1)
    want_h = dm.forward_hidden(tok)
    got_h = tp.forward_hidden(tok)
    assert np.array_equal(_bits(got_h), _bits(want_h))
    s_ref = dm.new_states(2)
    dm.prefill(tok, s_ref)
    s_tp = tp.new_states(2)
    tp.prefill(tok, s_tp)
    cur = tok[:, -1].contiguous()
    for _ in range(3):
        a = dm.decode_step(cur, s_ref)
        b = tp.decode_step(cur, s_tp)
        assert np.array_equal(_bits(a), _bits(b))
        cur = a.argmax(-1)


def test_tp_model_graph_nccl(cuda):
    """The TP decode step with real NCCL collectives captured in a CUDA graph
    (one rank: the single-GPU box), replays bit-identical to DeviceModel's decode."""
    here = Path(__file__).resolve().parent
    port = str(29700 + os.getpid() % 1000)
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=port)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
                        "--master-addr", "127.0.0.1", "--master-port", port, str(here / "tp_nccl_worker.py")],
                       env=env, capture_output=True, text=True, timeout=600, cwd=str(here.parent))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "tp graph rank ok" in r.stdout, r.stdout[-2000:]
