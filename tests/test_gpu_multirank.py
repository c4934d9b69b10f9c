"""The GPU engine with 2 and 3 ranks (processes) on one B200, talking through
gloo (device buffers staged via the host).  No kernel waits on another rank:
every exchange is a host-side p2p.  Same iterations / history / solution as
one rank, and as the reference engine's fixture (worker-count invariance,
reference test_acceptance.py:229-267)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir, name, inner):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    from conftest import load_golden
    from paper_1912_03106_b200 import (CycleSpec, DistTransport, GpuFemProblem, MgritSolver,
                                       StoppingCriterion, TimeHierarchy, build_uniform_grid)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load_golden(name)
        spec = fx["spec"]
        mg = spec["mgrit"]
        prob = GpuFemProblem(spec, device=0, inner=inner)
        grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
        solver = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                             CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                       max_iters=int(fx["max_iters"]),
                                       spatial_strategy=mg["spatial_strategy"],
                                       nested_iterations=mg.get("nested_iterations", False)),
                             StoppingCriterion(tolerance=float(fx["tol"])),
                             DistTransport(device=torch.device("cuda", 0)))
        run, sol = solver.solve(gather_solution=True)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"),
                 hist=np.array([run.initial_residual] + run.residual_norms),
                 iters=run.iterations,
                 sol=sol.cpu().numpy() if sol is not None else np.zeros(0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name", ["mgrit_cfg2_delayed_n32", "mgrit_cfg2_nested_n32"])
def test_gpu_engine_worker_count_invariance(cuda, tmp_path, world, name):
    fx = load_golden(name)
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), name, "cholesky"),
             nprocs=world, join=True)
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for r in ranks:
        assert int(r["iters"]) == int(fx["iterations"])
        np.testing.assert_allclose(r["hist"], fx["history"], rtol=1e-8)
    m = int(fx["factors"][0])
    sol_c = ranks[0]["sol"][::m]
    assert np.linalg.norm(sol_c - fx["sol_c"]) / np.linalg.norm(fx["sol_c"]) < 1e-9


def _nccl_worker(rank, world, port, out_dir, name):
    """One rank, backend NCCL: the device-tensor branch of DistTransport
    (no host staging) -- collectives on a 1-rank communicator, a grouped
    isend/irecv pair to itself (ncclGroupStart/End), and a full solve."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch
    import torch.distributed as dist
    from conftest import load_golden
    from paper_1912_03106_b200 import (CycleSpec, DistTransport, GpuFemProblem, MgritSolver,
                                       StoppingCriterion, TimeHierarchy, build_uniform_grid)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    try:
        T = DistTransport(device=dev)
        assert not T.stage and T.coll_device == dev
        assert T.sum_ordered(1.25) == 1.25 and T.max(-3.0) == -3.0
        T.barrier()
        a = torch.arange(1000, dtype=torch.float64, device=dev)
        b = torch.zeros_like(a)
        h = T.exchange_async([(0, a)], [(0, b)])      # self-loop through the NCCL p2p path
        c = a * 2.0                                    # independent work while in flight
        h.wait()
        torch.cuda.synchronize(dev)
        assert torch.equal(a, b) and torch.equal(c, a * 2.0)
        fx = load_golden(name)
        spec = fx["spec"]
        mg = spec["mgrit"]
        prob = GpuFemProblem(spec, device=0, inner="cholesky")
        grid = build_uniform_grid(0.0, spec["tf"], spec["n_steps"])
        solver = MgritSolver(prob, TimeHierarchy.build(grid, mg["factors"]),
                             CycleSpec(kind=mg["kind"], gamma=mg["gamma"],
                                       max_iters=int(fx["max_iters"]),
                                       spatial_strategy=mg["spatial_strategy"]),
                             StoppingCriterion(tolerance=float(fx["tol"])), T)
        run, sol = solver.solve(gather_solution=True)
        np.savez(os.path.join(out_dir, "nccl.npz"),
                 hist=np.array([run.initial_residual] + run.residual_norms),
                 iters=run.iterations, sol=sol.cpu().numpy())
    finally:
        dist.destroy_process_group()


def test_nccl_transport_on_one_gpu(cuda, tmp_path):
    """The NCCL data plane (device tensors, grouped p2p, all-gather /
    all-reduce) on the one GPU a test box has: a 1-rank communicator.  The
    2..8-rank layout is covered by the gloo tests above and in
    test_multirank.py; this one proves the NCCL code path itself runs."""
    name = "mgrit_cfg2_delayed_n32"
    fx = load_golden(name)
    mp.spawn(_nccl_worker, args=(1, _free_port(), str(tmp_path), name), nprocs=1, join=True)
    r = np.load(tmp_path / "nccl.npz")
    assert int(r["iters"]) == int(fx["iterations"])
    np.testing.assert_allclose(r["hist"], fx["history"], rtol=1e-8)
    m = int(fx["factors"][0])
    sol_c = r["sol"][::m]
    assert np.linalg.norm(sol_c - fx["sol_c"]) / np.linalg.norm(fx["sol_c"]) < 1e-9
