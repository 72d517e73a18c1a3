"""Expert-parallel host logic with real collectives on CPU (gloo, world size 2 and 4): the count
exchange (C1), split sizes, source-major segment table and both all-to-alls of paper_2410_19123_b200.ep,
with the oracle standing in for the GPU kernels on each rank. The composed layer must equal the
single-process oracle bit for bit (P12)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, H, E, d, k, skew, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_2410_19123_b200 import ep
        El = E // world
        x = synth.tokens(T * world, H, seed=1)
        if skew:
            lg = synth.logits_for_assignments(synth.assignments_zipf(T * world, E, 1.0, seed=2), E, seed=2)
        else:
            lg = synth.router_logits(T * world, E, seed=2)
        wg, wu, wd = synth.expert_weights(E, d, H, seed=3)
        xl, ll = x[rank * T:(rank + 1) * T], lg[rank * T:(rank + 1) * T]
        plan = oracle.route(ll, k)
        ep_plan = ep.plan_from_counts(torch.from_numpy(plan["counts"].astype(np.int32)))
        assert sum(ep_plan.send_splits) == T * k
        xs = torch.from_numpy(oracle.dispatch(xl, plan["dest"], k))
        x_recv = ep.exchange(xs, ep_plan)
        assert x_recv.shape[0] == ep_plan.rows_in
        sl = slice(rank * El, (rank + 1) * El)
        y_recv = oracle.expert_ffn(x_recv.numpy(), ep_plan.seg_offsets.astype(np.int32), wg[sl], wu[sl], wd[sl],
                                   n_src=world)
        ys = ep.exchange(torch.from_numpy(y_recv), ep_plan, reverse=True)
        y = oracle.combine(ys.numpy(), plan["dest"], plan["topk_w"], k)
        ref, _ = oracle.moe_layer(x, lg, k, wg, wu, wd)
        q.put((rank, bool(np.array_equal(y, ref[rank * T:(rank + 1) * T])), ep_plan.recv_splits))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,E,k,skew", [(2, 96, 8, 1, False), (2, 64, 8, 2, True), (4, 48, 8, 1, True)])
def test_ep_gloo_equals_single_layer(world, T, E, k, skew):
    H, d = 16, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, H, E, d, k, skew, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, splits in res:
        assert ok is True, f"rank {rank}: {ok}"
