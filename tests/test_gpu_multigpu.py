"""World-size-2 NCCL run of the sharded multi-GPU paths on the CUDA library:
config-4-style batched E / grad E sharded by latent column and the order-2 Lipschitz loss
sharded by pair (paper_2409_03807_b200/replicas.py), one process per GPU.  Each rank's shard
runs through lsb_eval_batched / lsb_lipschitz_loss on its own device; the gathered results
must equal a single-GPU run of the whole batch.  Skipped on boxes with fewer than 2 GPUs
(the round-end driver and gpurun use one)."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


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
    import torch
    import torch.distributed as dist
    from paper_2409_03807_b200 import configs, replicas

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    pr = configs.build("c1")
    sysm = pr.system("fp32", device=rank)
    sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
    Z = configs.latent_batch_c4(pr.model.r, 96)
    E, G = replicas.sharded_eval(sysm.eval_batched, Z, dist, device=f"cuda:{rank}")
    sysm.set_inertia(None, configs.DT)
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 6)
    loss = replicas.sharded_lipschitz_loss(lambda a, b: sysm.lipschitz_loss(a, b) * a.shape[0], Z1, Z2, dist,
                                           device=f"cuda:{rank}")
    t = replicas.max_over_ranks(1.0 + rank, dist, device=f"cuda:{rank}")
    out[rank] = (E, G, loss, t)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(_gpus() < 2, reason="needs 2 GPUs (world size 2, one process per GPU)")
def test_sharded_batched_eval_and_loss_on_two_gpus(product):
    import multiprocessing as mp
    from paper_2409_03807_b200 import configs
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    pr = configs.build("c1")
    sysm = pr.system("fp32")
    sysm.set_inertia(configs.timestep0_qbar(pr, sysm.mass), configs.DT)
    Z = configs.latent_batch_c4(pr.model.r, 96)
    E_ref, G_ref = sysm.eval_batched(Z)
    sysm.set_inertia(None, configs.DT)
    Z1, Z2 = configs.latent_pairs_c5(pr.model.r, 6)
    loss_ref = sysm.lipschitz_loss(Z1, Z2)
    for r in range(2):
        E, G, loss, t = out[r]
        # per-column results do not depend on the batch split (column-independent kernels)
        assert np.allclose(E, E_ref, rtol=1e-12, atol=0) and np.allclose(G, G_ref, rtol=1e-10, atol=1e-14)
        assert abs(loss - loss_ref) <= 1e-10 * abs(loss_ref)
        assert t == 2.0
