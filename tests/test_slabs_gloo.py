"""Multi-rank (world_size 2 and 3) host logic on CPU with the gloo backend:
the engine's own slab plan (po_slab_plan, the C++ partition Engine::Engine
uses, called here through the C ABI without a GPU), the halo exchange with the
peers that plan names, the Gram all-reduce and the RHS all-gather reproduce the
single-domain oracle."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, size, port_num, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_num)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import port
        from paper_1510_07230_b200 import configs, native, slabs

        spec = configs.ProblemSpec("gl", (11, 6, 7), (5.0, 4.0, 4.5), [], 3, hartree=False, xc=False)
        rng = np.random.default_rng(11)
        u = rng.standard_normal((3, spec.num_points))
        plane = spec.n[1] * spec.n[2]
        z0, nz, lo_peer, hi_peer = native.slab_plan(spec.n[0], size, rank)  # the engine's C++ plan
        assert (z0, nz) == slabs.slab_bounds(spec.n[0], size, rank)
        assert lo_peer == (rank - 1 if rank > 0 else -1) and hi_peer == (rank + 1 if rank + 1 < size else -1)
        # the plans of all ranks tile the axis exactly (gathered over gloo)
        plans = [None] * size
        dist.all_gather_object(plans, (z0, nz))
        assert plans[0][0] == 0 and sum(p[1] for p in plans) == spec.n[0]
        assert all(plans[r][0] + plans[r][1] == plans[r + 1][0] for r in range(size - 1))
        ul = u[:, z0 * plane:(z0 + nz) * plane]
        lap = slabs.sharded_laplacian(ul, spec.n[1], spec.n[2], spec.spacing, rank, size, dist)
        want = np.stack([port.laplacian(spec, x) for x in u])[:, z0 * plane:(z0 + nz) * plane]
        err_lap = float(np.max(np.abs(lap - want)))
        g = slabs.sharded_gram(ul, ul, float(np.prod(spec.spacing)), dist)
        err_g = float(np.max(np.abs(g - port.gram(spec, u, u, same=True))))
        full = slabs.gather_full(ul[0].copy(), spec.n[0], plane, rank, size, dist)
        err_gather = float(np.max(np.abs(full - u[0])))
        q.put((rank, z0, nz, err_lap, err_g, err_gather))
    except Exception as ex:  # surfaced by the parent
        import traceback
        q.put((rank, "error", traceback.format_exc()[-1500:]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_slab_collectives_gloo(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_num = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port_num, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    errors = [r[2] for r in res if r[1] == "error"]
    assert not errors, errors[0]
    res.sort()
    assert sum(r[2] for r in res) == 11 and [r[1] for r in res] == sorted(r[1] for r in res)
    for _, _, _, e_lap, e_g, e_gather in res:
        assert e_lap < 1e-12 and e_g < 1e-13 and e_gather == 0.0


def test_slab_bounds_match_engine_partition(native):
    from paper_1510_07230_b200.slabs import slab_bounds

    with pytest.raises(native.InvalidArgument):
        native.slab_plan(3, 4, 0)  # fewer planes than ranks (po_create rejects it too)
    for n0 in (7, 64, 96, 128, 192):
        for size in (1, 2, 3, 4, 8):
            if n0 < size:
                continue
            spans = [slab_bounds(n0, size, r) for r in range(size)]
            assert spans == [native.slab_plan(n0, size, r)[:2] for r in range(size)]
            assert spans[0][0] == 0 and sum(nz for _, nz in spans) == n0
            assert all(spans[r][0] + spans[r][1] == spans[r + 1][0] for r in range(size - 1))
            assert max(nz for _, nz in spans) - min(nz for _, nz in spans) <= 1
