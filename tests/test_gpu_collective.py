"""The peer-memory all-reduce fused with the residual add
(ps_allreduce_add_bf16 / collective.P2PAllReduce):
x += sum over ranks of their bf16 partials, eagerly and from CUDA-graph
replays (device epochs), with one rank and with two ranks sharing the GPU
(separate processes, CUDA IPC mappings, gloo carrying only the handles)."""

import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

B, D = 16, 512


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial(rank, call):
    g = torch.Generator(device="cuda").manual_seed(1000 * rank + call)
    return torch.randn(B, D, device="cuda", generator=g).bfloat16()


def _run(ar, rank, world, calls, graph):
    """Returns (got, expected) residuals after `calls` all-reduces."""
    x = torch.randn(B, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(7))
    want = x.clone()
    for c in range(calls):
        for r in range(world):
            want += _partial(r, c).float()
    if not graph:
        for c in range(calls):
            ar.next_buffer((B, D)).copy_(_partial(rank, c))
            ar.add_into(x)
        torch.cuda.synchronize()
        return x, want
    # graph: the partial copies + all-reduces of `calls` calls, replayed with
    # the same inputs twice (epochs advance on the device)
    srcs = [_partial(rank, c) for c in range(calls)]
    x0 = x.clone()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        for c in range(calls):
            ar.next_buffer((B, D)).copy_(srcs[c])
            ar.add_into(x)
    torch.cuda.current_stream().wait_stream(st)
    for _ in range(2):
        x.copy_(x0)
        g.replay()
        torch.cuda.synchronize()
    return x, want


def test_p2p_allreduce_single_rank_eager_and_graph():
    from paper_2505_14884_b200.collective import P2PAllReduce

    ar = P2PAllReduce(None, 0, 1, B * D, "cuda")
    for graph in (False, True):
        got, want = _run(ar, 0, 1, 4, graph)
        assert float((got - want).abs().max()) <= 1e-4


def _rank(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2505_14884_b200.collective import P2PAllReduce

        ar = P2PAllReduce(dist.group.WORLD, rank, world, B * D, "cuda")
        errs = []
        for graph in (False, True):
            dist.barrier()
            got, want = _run(ar, rank, world, 3, graph)
            errs.append(float((got - want).abs().max()))
        dist.barrier()
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


def test_p2p_allreduce_two_ranks_share_the_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = dict(q.get(timeout=10) for _ in range(2))
    for r in range(2):
        assert max(res[r]) <= 1e-4, res
