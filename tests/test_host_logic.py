"""CPU tests of the host-side logic: the reference's controller arithmetic
(against reference-generated values and the reference's own known answers),
the ActivationStore lifecycle, the layer map, and the cross-rank statistics
sync (gloo, world size 2)."""
import math
import os

import numpy as np
import pytest

from paper_2111_09562_b200 import controller as ctl
from paper_2111_09562_b200.errors import LifecycleError, MemoryInfeasibleError, ParameterError
from paper_2111_09562_b200.hooks import ActivationCompressor, ActivationStore, sync_layer_stats


def stats(layer_id="conv1", R=0.5, L_bar=2.0, M_avg=1.0, N=64, **kw):
    return ctl.LayerTrainingStats(layer_id=layer_id, R=R, L_bar=L_bar, M_avg=M_avg, N=N, **kw)


def plan_of(eb_map, W=1000, interval=1):
    return ctl.CompressionPlan(eb=eb_map, W=W, interval_index=interval, skip=frozenset())


def test_hand_computed_eb():
    # reference test_controller.py:101-105
    plan = ctl.plan_compression([stats()], ctl.ControllerConfig())
    assert plan.eb["conv1"] == pytest.approx(2.7621358640099365e-3, rel=1e-12)


def test_eb_matches_reference_golden(golden_meta):
    s = golden_meta["stats"]
    st = ctl.LayerTrainingStats("conv1", R=s["collect"]["R"], L_bar=s["collect"]["L_bar"], M_avg=s["collect"]["M_avg"], N=8)
    assert ctl.plan_compression([st], ctl.ControllerConfig()).eb["conv1"] == s["plan_eb"]


def test_estimate_eb_inverse():
    for a, L, N, R, eb in [(0.32, 2.0, 64, 0.5, 1e-3), (0.1, 0.3, 7, 0.9, 3e-5)]:
        sig = ctl.predict_sigma(a, L, N, R, eb)
        assert ctl.estimate_eb(sig, a, L, N, R) == pytest.approx(eb, rel=1e-14)
    assert ctl.estimate_eb(1.0, 0.32, 0.0, 8, 0.5) is None
    assert ctl.estimate_eb(1.0, 0.32, 1.0, 8, 0.0) is None


def test_update_interval_cases():
    # reference test_controller.py:144-197
    cfg = ctl.ControllerConfig()
    assert ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 2.5e-3}), 1000, cfg) == (500, 0)
    assert ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 2e-3}), 1000, cfg)[0] == 1000
    assert ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 1e-3 / 2.5}), 1000, cfg)[0] == 500
    W, k = ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 1.1e-3}), 250, cfg, 0)
    assert (W, k) == (250, 1)
    assert ctl.update_interval(plan_of({"c": 1.1e-3}), plan_of({"c": 1e-3}), W, cfg, k) == (1000, 0)
    W = 250
    for _ in range(4):
        W, _ = ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 1e-1}), W, cfg)
    assert W == 125
    assert ctl.update_interval(None, plan_of({"c": 1e-3}), 1000, cfg) == (1000, 0)
    assert ctl.update_interval(plan_of({"c": 1e-3}), plan_of({"c": 1.5e-3}), 500, cfg, 1) == (500, 0)


def test_skip_and_validation():
    plan = ctl.plan_compression([stats("a", R=0.0), stats("b", M_avg=0.0), stats("c")], ctl.ControllerConfig())
    assert plan.skip == frozenset({"a", "b"}) and set(plan.eb) == {"c"}
    with pytest.raises(ParameterError):
        ctl.LayerTrainingStats("x", R=1.5, L_bar=1.0, M_avg=1.0, N=1)
    with pytest.raises(ParameterError):
        ctl.CompressionPlan(eb={"x": 0.0}, W=10, interval_index=0, skip=frozenset())


def test_batch_planner():
    cfg = ctl.ControllerConfig(memory_budget_bytes=10 ** 9)
    b = ctl.choose_batch_size({"l1": 1e6, "l2": 2e6}, {"l1": 4.0, "l2": 8.0}, cfg)
    assert b == 1024 or b * (1e6 / 4 + 2e6 / 8) <= 10 ** 9 * 0.95
    with pytest.raises(MemoryInfeasibleError):
        ctl.choose_batch_size({"l1": 1e12}, {}, cfg)


def test_adaptive_controller_W():
    cfg = ctl.ControllerConfig(W_default=8, W_floor=2)
    c = ctl.AdaptiveController(cfg)
    p1 = c.new_interval([stats(M_avg=1.0)])
    p2 = c.new_interval([stats(M_avg=3.0)])  # eb x3 -> halve W
    assert p1.W == 8 and p2.W == 4 and c.intervals_planned == 2


def test_activation_store_lifecycle():
    s = ActivationStore()
    s.put("conv1", ActivationStore.COMPRESSED, object(), 100)
    s.put("conv2", ActivationStore.RAW, object(), 400)
    assert s.current_bytes == 500 and s.peak_bytes == 500
    with pytest.raises(LifecycleError):
        s.put("conv1", ActivationStore.RAW, None, 1)
    kind, _, nb = s.pop("conv1")
    assert kind == ActivationStore.COMPRESSED and nb == 100 and s.current_bytes == 400
    with pytest.raises(LifecycleError):
        s.pop("conv1")


def _trace(model, x, iters=1):
    """run the hooks in passthrough mode (first interval: slots filled raw,
    no codec) on the CPU -- exercises the slot / consumer dataflow"""
    torch = pytest.importorskip("torch")

    opt = torch.optim.SGD(model.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(model), opt,
                                ctl.ControllerConfig(W_default=1000, W_floor=1))
    y = torch.zeros(x.shape[0], dtype=torch.long)
    for _ in range(iters):
        opt.zero_grad()
        with comp.iteration():
            out = model(x)
            torch.nn.functional.cross_entropy(out, y[: out.shape[0]]).backward()
        opt.step()
        comp.after_step()
        assert comp.store.current_bytes == 0 and len(comp.store) == 0  # every slot consumed once
    return comp


def test_conv_layer_map_sequential():
    torch = pytest.importorskip("torch")
    import torch.nn as nn

    torch.manual_seed(0)
    net = nn.Sequential(nn.Conv2d(3, 8, 3), nn.ReLU(inplace=True), nn.MaxPool2d(2), nn.Conv2d(8, 8, 3), nn.ReLU(),
                        nn.Flatten(), nn.Linear(8 * 4 * 4, 4))
    m = ActivationCompressor.conv_layer_map(net)
    assert list(m) == ["0", "3"] and m.model is net
    comp = _trace(net, torch.randn(2, 3, 14, 14), iters=2)
    r = comp.records[-1]
    assert r.slots == ["0", "3"] and r.markers == 1  # the max-pool output is recomputed
    assert comp.consumer_names() == {"0": "3", "3": "6"}  # through a Flatten module
    assert net[1].inplace


def test_dataflow_slots_resnet50():
    """torchvision Bottleneck calls one ReLU module three times per block:
    each call is its own slot (the conv it follows); conv3's consumer is the
    next block's conv1 across the residual add, not downsample.0 (reference
    _consumer_map semantics, training.py:154-166)."""
    torch = pytest.importorskip("torch")
    tv = pytest.importorskip("torchvision")

    torch.manual_seed(0)
    net = tv.models.resnet50(num_classes=10)
    comp = _trace(net, torch.randn(2, 3, 64, 64), iters=2)
    r = comp.records[-1]
    convs = [n for n, mod in net.named_modules() if isinstance(mod, torch.nn.Conv2d) and "downsample" not in n]
    assert r.slots == convs and len(r.slots) == 49
    cn = comp.consumer_names()
    assert cn["conv1"] == "layer1.0.conv1"  # through the stem max-pool
    assert cn["layer1.0.conv3"] == "layer1.1.conv1" and cn["layer1.2.conv3"] == "layer2.0.conv1"
    assert cn["layer2.0.conv1"] == "layer2.0.conv2" and cn["layer4.2.conv3"] == "fc"
    # the ReLU after conv -> BN (stem, conv1 and conv2 of every block) is
    # recomputed from the stored conv output; conv3's ReLU follows a residual
    # add and stays stored; plus the stem max-pool (read by layer1.0.conv1
    # and downsample.0)
    assert r.markers == 1 + 2 * 16 + 1


def test_dataflow_slots_vgg16_alexnet():
    torch = pytest.importorskip("torch")
    tv = pytest.importorskip("torchvision")

    torch.manual_seed(0)
    vgg = tv.models.vgg16(num_classes=10)
    comp = _trace(vgg, torch.randn(2, 3, 32, 32))
    r = comp.records[-1]
    assert len(r.slots) == 13 and r.markers == 5
    assert comp.consumer_names()["features.28"] == "classifier.0"
    alex = tv.models.alexnet(num_classes=10)
    comp = _trace(alex, torch.randn(2, 3, 96, 96))
    assert comp.consumer_names() == {"features.0": "features.3", "features.3": "features.6",
                                     "features.6": "features.8", "features.8": "features.10",
                                     "features.10": "classifier.1"}


def test_shared_modules_get_per_call_slots():
    """a conv called twice and a ReLU module shared by two convs: one slot
    per call, no LifecycleError"""
    torch = pytest.importorskip("torch")
    import torch.nn as nn

    class Net(nn.Module):
        def __init__(self):
            super().__init__()
            self.a = nn.Conv2d(4, 4, 3, padding=1)
            self.b = nn.Conv2d(4, 4, 3, padding=1)
            self.relu = nn.ReLU(inplace=True)
            self.fc = nn.Linear(4 * 8 * 8, 3)

        def forward(self, x):
            x = self.relu(self.a(x))
            x = self.relu(self.a(x))
            x = self.relu(self.b(x))
            return self.fc(torch.flatten(x, 1))

    torch.manual_seed(0)
    net = Net()
    comp = _trace(net, torch.randn(2, 4, 8, 8), iters=2)
    assert comp.records[-1].slots == ["a", "a#1", "b"]
    assert comp.consumer_names() == {"a": "a", "a#1": "b", "b": "fc"}


def test_compressor_batch_planner_and_reserve_breaches():
    """ActivationCompressor's memory-budget planner (reference training.py:
    401-426): per-sample layer costs / interval ratios + fixed model bytes
    -> choose_batch_size; store peak + fixed over the usable budget counts
    a reserve breach."""
    torch = pytest.importorskip("torch")
    import torch.nn as nn

    net = nn.Sequential(nn.Conv2d(3, 8, 3), nn.ReLU(), nn.Conv2d(8, 8, 3), nn.ReLU(), nn.Flatten(), nn.Linear(8, 4))
    opt = torch.optim.SGD(net.parameters(), lr=0.1, momentum=0.9)
    cfg = ctl.ControllerConfig(memory_budget_bytes=10 ** 6, reserve_fraction=0.1)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(net), opt, cfg, input_sample_bytes=3 * 32 * 32 * 4)
    nparams = sum(p.numel() for p in net.parameters())
    assert comp.fixed_bytes == 2 * 4 * nparams  # weights + velocity, fp32 (training.py:200)
    comp._per_sample = {"0": 8 * 30 * 30 * 4.0, "2": 8 * 28 * 28 * 4.0}  # per stored slot
    comp._interval_ratios = {"0": [4.0, 6.0], "2": [8.0]}
    want = ctl.choose_batch_size({"input": 3 * 32 * 32 * 4.0, "0": 8 * 30 * 30 * 4.0, "2": 8 * 28 * 28 * 4.0},
                                 {"0": 5.0, "2": 8.0}, cfg, fixed_bytes=comp.fixed_bytes)
    assert comp.plan_batch_size() == want
    per_b = 3 * 32 * 32 * 4 + 8 * 30 * 30 * 4 / 5 + 8 * 28 * 28 * 4 / 8
    assert want * per_b + comp.fixed_bytes <= 0.9 * 10 ** 6 < 2 * want * per_b + comp.fixed_bytes
    # reserve breach accounting on after_step
    comp._rec = None
    comp.store.peak_bytes = 10 ** 6
    comp.after_step()
    comp.store.peak_bytes = 0
    comp.after_step()
    assert comp.reserve_breaches == 1 and comp.it == 2


def _sync_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    R, L, M = sync_layer_stats([0.5 + 0.1 * rank, 0.2], [1.0 * (rank + 1), 0.0], [0.01, 0.02])
    plan = ctl.plan_compression([ctl.LayerTrainingStats(f"c{i}", R=R[i], L_bar=L[i], M_avg=M[i], N=16)
                                 for i in range(2)], ctl.ControllerConfig())
    q.put((rank, R, L, M, dict(plan.eb), sorted(plan.skip)))
    dist.destroy_process_group()


def test_stats_sync_two_ranks_gloo():
    """world_size 2 on gloo: both ranks see averaged stats and identical eb."""
    import multiprocessing as mp
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_sync_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    (_, R0, L0, M0, eb0, sk0), (_, R1, L1, M1, eb1, sk1) = res
    assert R0 == R1 == [pytest.approx(0.55), pytest.approx(0.2)]
    assert L0 == L1 == [pytest.approx(1.5), 0.0]
    assert eb0 == eb1 and sk0 == sk1 == ["c1"]


def test_marker_recompute_gives_identical_gradients():
    """MARKER slots (pooling outputs recomputed in backward from the stored
    activation, training.py:295-296, 344-347) change no value: with the
    stored activations raw (first interval), every parameter gradient equals
    that of the same step without the hooks, bit for bit."""
    torch = pytest.importorskip("torch")
    import torch.nn as nn

    def net():
        torch.manual_seed(3)
        return nn.Sequential(nn.Conv2d(3, 8, 3), nn.ReLU(inplace=True), nn.MaxPool2d(2), nn.Conv2d(8, 8, 3),
                             nn.ReLU(), nn.AvgPool2d(2), nn.Conv2d(8, 6, 1), nn.ReLU(), nn.Flatten(),
                             nn.Linear(6 * 2 * 2, 4))

    x = torch.randn(4, 3, 14, 14, generator=torch.Generator().manual_seed(5))
    y = torch.tensor([0, 1, 2, 3])
    ref = net()
    torch.nn.functional.cross_entropy(ref(x), y).backward()
    hooked = net()
    opt = torch.optim.SGD(hooked.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(hooked), opt,
                                ctl.ControllerConfig(W_default=1000, W_floor=1))
    with comp.iteration():
        torch.nn.functional.cross_entropy(hooked(x), y).backward()
    grads = [p.grad.clone() for p in hooked.parameters()]
    opt.step()
    comp.after_step()
    assert comp.records[-1].markers == 2  # max-pool and avg-pool outputs recomputed
    for (n, _), g, q in zip(hooked.named_parameters(), grads, ref.parameters()):
        assert torch.equal(g, q.grad), n


def test_bn_relu_recompute_matches_plain_step():
    """conv -> BatchNorm -> ReLU: the stored activation is the conv output
    (BN's saved input) and the ReLU output is recomputed in backward with the
    forward pass's batch statistics (training.py:344-347).
    With raw storage (first interval) the step's gradients equal those of the
    plain step up to the recompute's rounding; after a residual add the ReLU
    output stays stored."""
    torch = pytest.importorskip("torch")
    import torch.nn as nn

    class Net(nn.Module):
        def __init__(self):
            super().__init__()
            self.c1, self.b1 = nn.Conv2d(3, 8, 3, padding=1), nn.BatchNorm2d(8)
            self.c2, self.b2 = nn.Conv2d(8, 8, 3, padding=1), nn.BatchNorm2d(8)
            self.relu = nn.ReLU(inplace=True)
            self.pool = nn.MaxPool2d(2)
            self.fc = nn.Linear(8 * 4 * 4, 4)

        def forward(self, x):
            x = self.pool(self.relu(self.b1(self.c1(x))))
            y = self.b2(self.c2(x))
            y += x  # residual: the ReLU after it keeps its stored output
            return self.fc(torch.flatten(self.relu(y), 1))

    x = torch.randn(4, 3, 8, 8, generator=torch.Generator().manual_seed(7))
    y = torch.tensor([0, 1, 2, 3])
    torch.manual_seed(1)
    ref = Net()
    torch.nn.functional.cross_entropy(ref(x), y).backward()
    torch.manual_seed(1)
    hooked = Net()
    opt = torch.optim.SGD(hooked.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(hooked), opt,
                                ctl.ControllerConfig(W_default=1000, W_floor=1))
    with comp.iteration():
        torch.nn.functional.cross_entropy(hooked(x), y).backward()
    grads = [p.grad.clone() for p in hooked.parameters()]
    opt.step()
    comp.after_step()
    r = comp.records[-1]
    assert r.slots == ["c1", "c2"]
    assert r.markers == 2  # relu@c1 and the max-pool after it
    assert comp.store.current_bytes == 0
    for (n, _), g, q in zip(hooked.named_parameters(), grads, ref.parameters()):
        assert torch.allclose(g, q.grad, rtol=1e-4, atol=1e-6), n
