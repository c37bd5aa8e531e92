"""Multi-process (gloo, world size 2, CPU) tests of the image sharding and the
per-image result exchange used by bench.py at N > 1.  The
per-image numbers come from the oracle (the CUDA path needs a GPU); what is
tested here is the host-side partition + all-reduce logic."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_11651_b200 import dist as ccdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, per_rank, out_dir):
    import oracle
    import workload
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = workload.CONFIGS["tiny"].replace(H=24, W=40)
    owned = ccdist.owned_images(rank, per_rank)
    local = torch.zeros((per_rank, 4), dtype=torch.float64)
    for k, g in enumerate(owned):
        r = oracle.rd_forward_image(cfg, workload.make_image(cfg, workload.image_seed(7, g)))
        local[k] = torch.tensor([r["rate_bits"], r["sse"], r["mse"], r["cost"]])
    table = ccdist.allreduce_results(ccdist.scatter_results(local, rank, world, per_rank))
    mx = ccdist.max_over_ranks(float(rank + 1))
    np.save(os.path.join(out_dir, f"r{rank}.npy"), table.numpy())
    np.save(os.path.join(out_dir, f"m{rank}.npy"), np.array([mx]))
    dist.destroy_process_group()


def test_owned_images_partition():
    world, per = 4, 16
    seen = sorted(g for r in range(world) for g in ccdist.owned_images(r, per))
    assert seen == list(range(world * per))


@pytest.mark.timeout(300)
def test_gloo_world2_result_exchange(tmp_path):
    import oracle
    import workload
    world, per = 2, 3
    mp.spawn(_worker, args=(world, _free_port(), per, str(tmp_path)), nprocs=world, join=True)
    cfg = workload.CONFIGS["tiny"].replace(H=24, W=40)
    want = np.zeros((world * per, 4))
    for g in range(world * per):
        r = oracle.rd_forward_image(cfg, workload.make_image(cfg, workload.image_seed(7, g)))
        want[g] = [r["rate_bits"], r["sse"], r["mse"], r["cost"]]
    for rank in range(world):
        got = np.load(tmp_path / f"r{rank}.npy")
        np.testing.assert_array_equal(got, want)   # each row has one non-zero contributor: exact
        assert np.load(tmp_path / f"m{rank}.npy")[0] == world
