"""N = 2 over real NCCL (skipped on a 1-GPU box): request sharding with no data-path collective,
the int64 per-pair stats all-reduce, and G-invariance -- every rank's shard reproduces the
single-process run request by request, bit for bit, and the all-reduced stats equal the
single-process totals exactly on both ranks."""
import os
import socket
import tempfile

import pytest
import torch
import torch.multiprocessing as mp

pytestmark = [pytest.mark.gpu]

B, V = 16, 30000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(n, req0, dev):
    from paper_2505_07680_b200 import synth
    c = synth.CONFIGS["llama3"]
    return synth.gauss_chain(n, V, c["K"], c["L"], c["sigmas"], seed=c["seed"], req0=req0, device=dev, dtype="bf16")


def _rank(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world), RANK=str(rank),
                      LOCAL_RANK=str(rank))
    from paper_2505_07680_b200 import api
    from paper_2505_07680_b200 import dist as mdist
    torch.cuda.set_device(rank)
    mdist.init_from_env("nccl")
    r0, n = mdist.shard(B, world, rank, "strong")
    inp = _inputs(n, r0, f"cuda:{rank}")
    o = api.chain_verify(inp.levels, inp.draft, inp.u_acc, inp.u_emit, V=V)
    local = o["stats"].clone()
    mdist.allreduce_stats(o["stats"])
    torch.cuda.synchronize()
    torch.save({"r0": r0, "n": n, "local": local.cpu(), **{k: v.cpu() for k, v in o.items()}},
               os.path.join(out_dir, f"rank{rank}.pt"))
    torch.distributed.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_two_rank_nccl_shards_match_single_process():
    from paper_2505_07680_b200 import api
    full = _inputs(B, 0, "cuda:0")
    ref = {k: v.cpu() for k, v in api.chain_verify(full.levels, full.draft, full.u_acc, full.u_emit, V=V).items()}
    torch.cuda.synchronize()
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(2, _free_port(), d), nprocs=2, join=True)
        parts = [torch.load(os.path.join(d, f"rank{r}.pt")) for r in range(2)]
    for p in parts:
        sl = slice(p["r0"], p["r0"] + p["n"])
        for k in ("commit_tok", "commit_len", "flags"):
            assert torch.equal(p[k], ref[k][sl]), k
        for k in ("n_acc", "m_cand", "rollback", "pos_dtv", "pos_kl"):
            assert torch.equal(p[k], ref[k][:, sl]), k
        assert torch.equal(p["stats"], ref["stats"])             # all-reduced == single process
    assert torch.equal(parts[0]["local"] + parts[1]["local"], ref["stats"])
