"""The NCCL backend across processes: one process per GPU (torch.multiprocessing, NCCL id broadcast
through a gloo process group), X sliced into slabs along its last mode, every
exchange C1-C5 through ncclAllReduce / ncclAllGather on real peers.  The gathered result equals the
fp64 oracle at the north_star bar.  Needs >= 2 CUDA devices (skipped otherwise: the single-GPU
boxes of this build cover the same control flow through the loopback communicator,
tests/test_gpu_parity.py::test_loopback_multirank_hosvd, and the NCCL calls through a 1-rank
communicator, tests/test_gpu_nccl.py)."""
import os
import socket

import numpy as np
import pytest

import oracle
from gen import synth
from tests import _metrics as M

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, x, oms, q, algo, out_dir):
    import torch.distributed as dist

    from paper_2001_07124_b200 import api as P
    from paper_2001_07124_b200 import partition
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank)
    obj = [P.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    lo, hi = partition.slab_range(cfg.dims[-1], world, rank)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        h = P.Handle(stream=stream, nccl_id=obj[0], nranks=world, rank=rank)
        xs = torch.from_numpy(synth.to_device_layout(np.asfortranarray(x[..., lo:hi]))).cuda()
        loc = []
        for n, o in enumerate(oms):
            rows = partition.omega_rows(cfg.dims, n, lo, hi)
            o = o if rows is None else o[rows[0]:rows[0] + rows[1]]
            loc.append(torch.from_numpy(np.ascontiguousarray(o)).cuda())
        res = P.rtucker_hosvd(h, xs, cfg.ranks, cfg.p, q, loc, last_offset=lo, last_global=cfg.dims[-1])
        h.sync()
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), *[t.cpu().numpy() for t in res["Q"]],
                 G=P.core_to_numpy(res["G"]), err=res["err"].cpu().numpy())
        h.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("algo,q", [("hosvd", 0), ("hosvd", 1)])
def test_nccl_two_processes(tmp_path, algo, q):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 CUDA devices (one process per GPU)")
    import dataclasses

    import torch.multiprocessing as mp
    world = 2
    cfg = dataclasses.replace(synth.CONFIGS["cfg5"].scaled((96, 88, 80), (8, 8, 8), (8, 8, 8)), q=q)
    x = synth.make_tensor(cfg)
    oms = [synth.gaussian_omega(cfg, n) for n in range(3)]
    ref = oracle.hosvd(x, cfg.ranks, oms, q=q)
    mp.spawn(_worker, args=(world, _free_port(), cfg, x, oms, q, algo, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"r{r}.npz") for r in range(world)]
    qg = [outs[0]["arr_0"], outs[0]["arr_1"], np.concatenate([o["arr_2"] for o in outs], axis=0)]
    for n in range(3):
        assert M.orth(qg[n]) <= 1e-12
        assert M.subspace(qg[n], ref["Q"][n]) <= 1e-5, (n, M.subspace(qg[n], ref["Q"][n]))
    assert M.recon(outs[0]["G"], qg, ref["G"], ref["Q"]) <= 1e-5
    assert abs(outs[0]["err"][0] - ref["E"]) / ref["E"] <= 1e-5
    np.testing.assert_array_equal(outs[0]["G"], outs[1]["G"])      # the core is replicated bit for bit
