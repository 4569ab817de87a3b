"""Multi-process plumbing of the multi-GPU paths on ONE GPU, without any kernel that waits on another
rank (the profiling recipe forbids running mutually-waiting ranks as separate processes on one GPU):

* row slabs: two processes each create their rank of a
  KronCGSlab(emulate=False) -- workspace sizes, CUDA IPC export / import of the workspaces through a
  gloo all-gather, kron_cg_create_slab with the peer pointers -- then store into each other's
  workspace through the IPC mappings (kcg_slab_probe_put: peer stores only) and read back their own
  after a host barrier;
* face sharding: bench.py under torchrun with 2 ranks on the GPU (gloo for the
  host-side barrier / max), whole faces per rank, independent kernels.
The solve of the row-slab path itself (ranks spinning on each other's flags) is covered by the
one-launch emulation (tests/test_gpu_slab.py) and the gloo CPU protocol tests (test_sharding.py)."""

import json
import os
import socket
import subprocess
import sys

import pytest

from gpu_util import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA GPU")]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _slab_rank(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2204_08057_b200.kroncg import KronCGSlab
    from synth import make_patch
    from synth.problems import stack
    ps = [make_patch(6, 9, 3, seed=50 + i, tau="loguniform") for i in range(2)]
    st = stack(ps)
    hits = torch.from_numpy(np.random.default_rng(1).uniform(1, 4, (2, 64, 64)))
    ctx = KronCGSlab(6, st["A"], st["noise_prec"], st["tau"], st["kappa2"], world, emulate=False,
                     hits=hits, device="cuda:0")
    ctx.probe_put(1000.0)
    dist.barrier()
    got = ctx.probe_get()
    dist.barrier()
    res = {"rank": rank, "got": got, "rows": ctx.rows, "shape_Y": list(ctx.shape_Y)}
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    with open(out_path, "w") as f:
        json.dump(res, f)


def test_row_slab_ipc_plumbing_two_processes(tmp_path):
    import torch.multiprocessing as mp
    from paper_2204_08057_b200 import build
    build.build()
    world, port = 2, _free_port()
    outs = [str(tmp_path / f"r{r}.json") for r in range(world)]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_slab_rank, args=(r, world, port, outs[r])) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0, p.exitcode
    for r in range(world):
        with open(outs[r]) as f:
            res = json.load(f)
        assert res["got"] == [1000.0, 1001.0], res  # both ranks' peer stores landed in this workspace
        assert res["rows"] == 32 and res["shape_Y"] == [1, 2, 9, 32, 64]


def test_face_shard_bench_two_ranks_one_gpu():
    """bench.py's world > 1 path (face sharding, max-over-ranks timing) as 2 processes on one GPU."""
    from paper_2204_08057_b200 import build
    build.build()
    env = dict(os.environ, KCG_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "1", "--shard-only", "--e2e-steps", "1",
           "--no-cpu-baseline", "--no-slab-probe", "--no-lanczos", "--no-variance", "--no-pcg", "--no-kohler",
           "--no-hs"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "face-shard2"
    assert d["value"] > 0 and d["iterations_per_face_rank0"]
    assert d["true_rel_residual"] <= 5e-10
