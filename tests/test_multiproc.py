"""World-size-2 gloo tests of the multi-rank paths on CPU:
sharded Lipschitz loss and sharded batched evaluation equal the single-rank
results (the compute is the CPU oracle here; on B200 ranks it is the CUDA
library), and max-over-ranks timing."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist

    from oracle import pyoracle
    from paper_2409_03807_b200 import replicas

    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = pyoracle.Oracle.bar(3, 2, 1, 1.0, 0.4, 0.3, 0.0, 0, True)
    o.set_material(2.0, 1.0, 5.0)
    o.bar_decoder(2, 1, 6, 1, 3, 0.4)
    rng = np.random.default_rng(0)
    Z1, Z2 = rng.standard_normal((5, 2)), rng.standard_normal((5, 2))
    loss = replicas.sharded_lipschitz_loss(lambda a, b: o.lipschitz_loss2(a, b) * a.shape[0], Z1, Z2, dist)
    Z = rng.standard_normal((7, 2))
    E, G = replicas.sharded_eval(lambda Zl: o.eval_batch(Zl, qbar=None), Z, dist)
    t = replicas.max_over_ranks(1.0 + rank, dist)
    out[rank] = (loss, E, G, t)
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_paths_match_single_rank(oracle):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    o = oracle.Oracle.bar(3, 2, 1, 1.0, 0.4, 0.3, 0.0, 0, True)
    o.set_material(2.0, 1.0, 5.0)
    o.bar_decoder(2, 1, 6, 1, 3, 0.4)
    rng = np.random.default_rng(0)
    Z1, Z2 = rng.standard_normal((5, 2)), rng.standard_normal((5, 2))
    ref_loss = o.lipschitz_loss2(Z1, Z2)
    Z = rng.standard_normal((7, 2))
    ref_E, ref_G = o.eval_batch(Z, qbar=None)
    for r in range(2):
        loss, E, G, t = out[r]
        assert abs(loss - ref_loss) <= 1e-12 * abs(ref_loss)
        assert np.array_equal(E, ref_E) and np.array_equal(G, ref_G)
        assert t == 2.0


def test_shard_range_partitions():
    from paper_2409_03807_b200.replicas import shard_range
    for total in [0, 1, 7, 1024]:
        for world in [1, 2, 3, 8]:
            parts = [shard_range(total, world, r) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == total
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)
