"""Expert parallelism with the real CUDA kernels on ONE GPU (-m gpu): G ranks run as G processes sharing
cuda:0 over the gloo backend (NCCL refuses two ranks on one device). Each rank routes its own tokens,
exchanges rows with the all-to-alls of paper_2410_19123_b200.ep, runs readme_expert_ffn over the
(source rank, local expert) segments of its expert shard and combines. The result must equal the
single-GPU layer bit for bit (P12: rows reach their expert in global token order and no kernel splits K)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, H, E, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from paper_2410_19123_b200 import ep
        from paper_2410_19123_b200 import readme as rd
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        El = E // world
        x = synth.to_torch(synth.tokens(T * world, H, seed=1), "bf16").to(dev)
        lg = torch.from_numpy(synth.router_logits(T * world, E, seed=2)).to(dev)
        W = [synth.to_torch(w, "bf16").to(dev) for w in synth.expert_weights(E, d, H, seed=3)]
        y_full, _ = rd.moe_layer(x, *W, logits=lg)
        sl = slice(rank * El, (rank + 1) * El)
        layer = ep.EPMoELayer(x[rank * T:(rank + 1) * T].contiguous(), lg[rank * T:(rank + 1) * T].contiguous(),
                              W[0][sl].contiguous(), W[1][sl].contiguous(), W[2][sl].contiguous(), E, 1)
        y = layer.step()
        torch.cuda.synchronize()
        ok = torch.equal(y, y_full[rank * T:(rank + 1) * T])
        q.put((rank, bool(ok), layer.ep.recv_splits))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_on_one_gpu_equals_single_layer(world):
    T, H, E, d = 512, 256, 8, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, T, H, E, d, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, splits in res:
        assert ok is True, f"rank {rank}: {ok}"


# ---- the fused path: all-to-alls inside the kernels, over peer memory (readme_ep_*) -------------------

def _peer_worker(rank, world, port, T, H, E, d, k, residual, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layer = None
    try:
        import synth
        from paper_2410_19123_b200 import ep
        from paper_2410_19123_b200 import readme as rd
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        El = E // world
        x = synth.to_torch(synth.tokens(T * world, H, seed=11), "bf16").to(dev)
        lg = torch.from_numpy(synth.router_logits(T * world, E, seed=12)).to(dev)
        W = [synth.to_torch(w, "bf16").to(dev) for w in synth.expert_weights(E, d, H, seed=13)]
        y_full, _ = rd.moe_layer(x, *W, k=k, logits=lg, residual=x if residual else None)
        sl = slice(rank * El, (rank + 1) * El)
        layer = ep.PeerEPLayer(T, H, E, k, W[0][sl].contiguous(), W[1][sl].contiguous(), W[2][sl].contiguous(),
                               device=dev)
        mine = slice(rank * T, (rank + 1) * T)
        ok = True
        for rep in range(2):  # the second batch reuses the arena (flag generations advance)
            layer.x.copy_(x[mine])
            layer.route(lg[mine].contiguous())
            y = layer.layer(residual=residual)
            torch.cuda.synchronize()
            ok = ok and torch.equal(y, y_full[mine]) and int(layer.dev_status.item()) == 0
        # the whole batch (route + count exchange + layer) captured once and replayed: the phase epochs
        # live in device memory, so every replay synchronises afresh
        side = torch.cuda.Stream()
        with torch.cuda.stream(side):
            g = torch.cuda.CUDAGraph()
            lg_mine = lg[mine].contiguous()
            with torch.cuda.graph(g, stream=side):
                layer.route(lg_mine)
                y = layer.layer(residual=residual)
        for rep in range(3):
            layer.out.zero_()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            ok = ok and torch.equal(y, y_full[mine]) and int(layer.dev_status.item()) == 0
        q.put((rank, bool(ok), None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc(), None))
    finally:
        if layer is not None:
            try:
                layer.close()
            except Exception:
                pass
        dist.destroy_process_group()


@pytest.mark.parametrize("world,k,residual", [(2, 1, True), (4, 1, False), (2, 2, True)])
def test_peer_ep_on_one_gpu_equals_single_layer(world, k, residual):
    """G processes share cuda:0; their arenas are mapped into each other with CUDA IPC, rows move by
    stores from the dispatch kernel and from the down-projection epilogue, phases by system-scope flags.
    The output equals the single-GPU layer bit for bit (P12)."""
    T, H, E, d = 384, 256, 8, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, T, H, E, d, k, residual, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, _ in res:
        assert ok is True, f"rank {rank}: {ok}"


# ---- the NCCL branch: device all-to-alls on a real NCCL process group --------------------------------------

def _nccl_worker(port, T, H, E, d, k, q):
    """world_size 1 on NCCL (legal on one GPU): exercises the device all_to_all_single path of ep.exchange /
    ep.plan_from_counts (no host staging) and the peer-memory path's flag phases under an NCCL group."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    layer = None
    try:
        import synth
        from paper_2410_19123_b200 import ep
        from paper_2410_19123_b200 import readme as rd
        assert not ep._host_staged(None)
        x = synth.to_torch(synth.tokens(T, H, seed=21), "bf16").to(dev)
        lg = torch.from_numpy(synth.router_logits(T, E, seed=22)).to(dev)
        W = [synth.to_torch(w, "bf16").to(dev) for w in synth.expert_weights(E, d, H, seed=23)]
        y_full, _ = rd.moe_layer(x, *W, k=k, logits=lg)
        nccl = ep.EPMoELayer(x, lg, *W, E, k)
        y = nccl.step()
        torch.cuda.synchronize()
        ok = torch.equal(y, y_full)
        ok = ok and nccl.ep.send_splits == [T * k] and nccl.ep.recv_splits == [T * k]
        layer = ep.PeerEPLayer(T, H, E, k, *W, device=dev)
        layer.x.copy_(x)
        layer.route(lg)
        y2 = layer.layer(residual=False)
        torch.cuda.synchronize()
        ok = ok and torch.equal(y2, y_full) and int(layer.dev_status.item()) == 0
        q.put((bool(ok), None))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((traceback.format_exc(), None))
    finally:
        if layer is not None:
            try:
                layer.close()
            except Exception:
                pass
        dist.destroy_process_group()


@pytest.mark.parametrize("k", [1, 2])
def test_nccl_branch_world1_equals_single_layer(k):
    """The NCCL exchange (device all_to_all_single with split sizes) and the peer-memory path both run under an
    NCCL process group of one rank and reproduce the single-GPU layer bit for bit."""
    T, H, E, d = 1000, 256, 8, 256
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_port(), T, H, E, d, k, q))
    p.start()
    ok, _ = q.get(timeout=300)
    p.join(timeout=60)
    assert ok is True, ok
