"""Multi-rank partitioning on CPU: world_size 2 over gloo,
127.0.0.1 rendezvous.  The per-shard compute is the oracle (test
infrastructure, injected as the runner); what is under test is the
product's partitioning, table slicing and exchange logic
(paper_2512_15742_b200/sharding.py), which must reproduce the unsharded
reference forward bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2512_15742_b200 import sharding, synthetic


class OracleRunner:
    """Test infrastructure: the oracle as a rank-local runner on CPU tensors."""

    def __init__(self, runtime_layers):
        self.tables = [oracle.Tables.from_runtime(rl) for rl in runtime_layers]
        self.output_dim = self.tables[-1].out_dim

    def forward_dev(self, x, batch):
        import torch
        y, _ = oracle.port_forward(self.tables, x.cpu().numpy().astype(np.float64), batch)
        return torch.from_numpy(y).to(x.device)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _head():
    return synthetic.runtime_layers(synthetic.synthetic_head(dims=(24, 17, 3), k=40, grid=7, int8=True, seed=4))


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        gpu = case.startswith("gpu_")
        kind = case[4:] if gpu else case
        dev = torch.device("cuda", 0) if gpu else torch.device("cpu")
        if gpu:
            import paper_2512_15742_b200 as hq
            runner = lambda rl: sharding.DeviceRunner(hq.upload(rl, device=0), max_batch=8)  # noqa: E731
        else:
            runner = OracleRunner
        layers = _head()
        x = torch.from_numpy(synthetic.synthetic_inputs(5, 24, seed=3, grid=7)).to(dev)
        if kind == "batch":
            bs = sharding.BatchSharded(runner(layers), rank, world)
            y = bs.forward(x, 5, 24)
        elif kind == "columns":
            shard, tail = sharding.column_sharded_layers(layers, rank, world)
            cs = sharding.ColumnSharded(runner(shard), runner(tail), layers[0].header.out_dim, rank, world)
            y = cs.forward(x, 5)
        else:  # heads
            heads = [synthetic.runtime_layers(synthetic.synthetic_head(dims=(24, 9, 3), k=30, grid=7, int8=True,
                                                                       seed=50 + h)) for h in range(5)]
            lo, hi = sharding.shard_ranges(5, world)[rank]
            hs = sharding.HeadSharded([runner(heads[h]) for h in range(lo, hi)], 5, 3, rank, world)
            y = hs.forward(x if rank == 0 else torch.zeros_like(x), 5, 24)
        if gpu:
            assert y.is_cuda  # the result stays on the device
        q.put((rank, y.cpu().numpy().astype(np.float64).tobytes()))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return [np.frombuffer(out[r], np.float64) for r in range(world)]


def test_shard_ranges_cover_and_balance():
    for n in (0, 1, 5, 256, 13664):
        for w in (1, 2, 3, 8):
            r = sharding.shard_ranges(n, w)
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            sizes = [hi - lo for lo, hi in r]
            assert max(sizes) - min(sizes) <= 1


def test_column_slices_reassemble_the_layer_bitwise():
    layers = _head()
    x = synthetic.synthetic_inputs(4, 24, seed=9, grid=7)
    full = oracle.Tables.from_runtime(layers[0])
    want, _ = oracle.port_forward([full], x, 4)
    parts = []
    for lo, hi in sharding.shard_ranges(17, 3):
        t = oracle.Tables.from_runtime(sharding.column_slice_runtime(layers[0], lo, hi))
        y, _ = oracle.port_forward([t], x, 4)
        parts.append(y.reshape(4, hi - lo))
    assert np.array_equal(np.concatenate(parts, axis=1).ravel(), want)


@pytest.mark.parametrize("case", ["batch", "columns"])
def test_two_rank_partitioning_equals_unsharded_forward(case):
    _two_rank_equals_unsharded(case)


def _two_rank_equals_unsharded(case):
    layers = _head()
    x = synthetic.synthetic_inputs(5, 24, seed=3, grid=7)
    want, _ = oracle.port_forward([oracle.Tables.from_runtime(rl) for rl in layers], x, 5)
    ys = _run(case)
    for y in ys:  # every rank holds the whole result, bitwise the reference's
        assert np.array_equal(y, want)


def test_two_rank_head_sharding_broadcasts_features_and_gathers_heads():
    x = synthetic.synthetic_inputs(5, 24, seed=3, grid=7)
    want = []
    for h in range(5):
        rl = synthetic.runtime_layers(synthetic.synthetic_head(dims=(24, 9, 3), k=30, grid=7, int8=True, seed=50 + h))
        y, _ = oracle.port_forward([oracle.Tables.from_runtime(r) for r in rl], x, 5)
        want.append(y)
    ys = _run("heads")
    for y in ys:
        assert np.array_equal(y, np.concatenate(want))


# ---------------------------------------------------------------------------
# the product runner: two ranks (gloo) sharing the one GPU, DeviceRunner on
# cuda:0, device tensors end to end; exact mode would be bitwise, fast mode
# (the runner's default) is checked against the oracle's tolerance scale

def _device_runner_case(case):
    from helpers import assert_close
    layers = _head()
    x = synthetic.synthetic_inputs(5, 24, seed=3, grid=7)
    tables = [oracle.Tables.from_runtime(rl) for rl in layers]
    want, scale = oracle.port_forward_l1(tables, x, 5)
    for y in _run("gpu_" + case):
        assert_close(y, want, scale)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["batch", "columns"])
def test_two_rank_device_runner_partitioning(case):
    _device_runner_case(case)


@pytest.mark.gpu
def test_two_rank_device_runner_head_sharding():
    from helpers import assert_close
    x = synthetic.synthetic_inputs(5, 24, seed=3, grid=7)
    ys = _run("gpu_heads")
    for h in range(5):
        rl = synthetic.runtime_layers(synthetic.synthetic_head(dims=(24, 9, 3), k=30, grid=7, int8=True, seed=50 + h))
        want, scale = oracle.port_forward_l1([oracle.Tables.from_runtime(r) for r in rl], x, 5)
        for y in ys:
            assert_close(y.reshape(5, -1)[h], want, scale)
