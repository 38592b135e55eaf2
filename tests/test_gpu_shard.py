"""The sharded path with the matcher in it: two gloo ranks on the one B200,
each matching its strong_shard block of a 7-pair batch (device generator,
its own context), results gathered to rank 0 -- every plane equal to one
process matching the whole batch (no exchange on the data path,
so sharding cannot change a result)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
N, W, H = 7, 160, 120


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import paper_2205_03133_b200 as P
    from paper_2205_03133_b200.shard import gather_to_rank0, strong_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = strong_shard(N, rank, world)
    cfg = P.PipelineConfig.baseline(1)
    dl, dr = P.synth_batch_gpu(1, sh.count, seed0=sh.start, width=W, height=H)
    d = torch.empty((sh.count, H, W), dtype=torch.float64, device="cuda")
    v = torch.empty((sh.count, H, W), dtype=torch.uint8, device="cuda")
    with P.Matcher(cfg, W, H, sh.count) as m:
        m.run_device_u8(sh.count, W, H, 1, dl.data_ptr(), dr.data_ptr(),
                        {"disparity": d.data_ptr(), "disparity_valid": v.data_ptr()},
                        dtype=P.F64, focal=500.0, baseline=5.0)
        torch.cuda.synchronize()
    # equal shapes for the gather: pad the shorter block with a copy of pair 0
    n_max = -(-N // world)
    dd = np.concatenate([d.cpu().numpy()] + [d[:1].cpu().numpy()] * (n_max - sh.count))
    vv = np.concatenate([v.cpu().numpy()] + [v[:1].cpu().numpy()] * (n_max - sh.count))
    gd, gv = gather_to_rank0(dd), gather_to_rank0(vv)
    counts = gather_to_rank0(np.array([sh.count]))
    if rank == 0:
        q.put((gd, gv, counts))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_match_like_one(gpu):
    P = gpu
    import torch

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gd, gv, counts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n_max = gd.shape[0] // 2
    parts_d = [gd[r * n_max: r * n_max + int(counts[r])] for r in range(2)]
    parts_v = [gv[r * n_max: r * n_max + int(counts[r])] for r in range(2)]
    dl, dr = P.synth_batch_gpu(1, N, seed0=0, width=W, height=H)
    with P.Matcher(P.PipelineConfig.baseline(1), W, H, N) as m:
        one = m.run_batch(dl.cpu().numpy(), dr.cpu().numpy(), focal=500.0, baseline=5.0,
                          dtype=P.F64, want=("disparity", "disparity_valid"))
    torch.cuda.synchronize()
    assert np.array_equal(np.concatenate(parts_v), one["disparity_valid"])
    assert np.array_equal(np.concatenate(parts_d).view(np.uint64), one["disparity"].view(np.uint64))
