"""GPU: training with compressed activations through saved_tensors_hooks."""
import math

import numpy as np

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import paper_2111_09562_b200 as pb  # noqa: E402
from paper_2111_09562_b200.hooks import ActivationCompressor  # noqa: E402


def _net():
    nn = torch.nn
    torch.manual_seed(0)
    return nn.Sequential(nn.Conv2d(3, 32, 3, padding=1), nn.ReLU(), nn.MaxPool2d(2),
                         nn.Conv2d(32, 64, 3, padding=1), nn.ReLU(), nn.MaxPool2d(2),
                         nn.Conv2d(64, 64, 3, padding=1), nn.ReLU(),
                         nn.Flatten(), nn.Linear(64 * 8 * 8, 10)).cuda()


def _run(compress, iters=8, budget=None):
    net = _net()
    opt = torch.optim.SGD(net.parameters(), lr=0.01, momentum=0.9)
    comp = None
    if compress:
        comp = ActivationCompressor(ActivationCompressor.conv_layer_map(net), opt,
                                    pb.ControllerConfig(W_default=2, W_floor=1, memory_budget_bytes=budget),
                                    input_sample_bytes=3 * 32 * 32 * 4)
    g = torch.Generator(device="cuda").manual_seed(1)
    losses = []
    for it in range(iters):
        x = torch.randn(16, 3, 32, 32, device="cuda", generator=g)
        y = torch.randint(0, 10, (16,), device="cuda", generator=g)
        opt.zero_grad()
        if comp:
            with comp.iteration():
                loss = torch.nn.functional.cross_entropy(net(x), y)
                loss.backward()
        else:
            loss = torch.nn.functional.cross_entropy(net(x), y)
            loss.backward()
        opt.step()
        if comp:
            comp.after_step()
        losses.append(float(loss))
    return net, comp, losses


def test_training_with_compression_engages_and_tracks_baseline():
    base, _, lb = _run(False)
    net, comp, lc = _run(True)
    assert all(math.isfinite(v) for v in lc)
    # first interval (W=2) is passthrough: identical losses
    assert lc[:2] == lb[:2]
    assert comp.plan is not None and set(comp.plan.eb) | set(comp.plan.skip) == set(comp.layers)
    later = [r for r in comp.records[2:] if r.compressed]
    assert later, "no layer was compressed after the first interval"
    for r in later:
        assert r.stored_bytes < r.raw_bytes
        for lid, (ratio, eb) in r.compressed.items():
            assert ratio > 1.0 and eb > 0
    # bounded activation error -> the weights stay close to the baseline run
    for pc, pbse in zip(net.parameters(), base.parameters()):
        rel = (pc - pbse).norm() / (pbse.norm() + 1e-12)
        assert rel < 0.05, float(rel)


def test_hooks_handle_shared_saved_tensors():
    # ReLU output saved by both relu backward and maxpool -> compressed once, unpacked twice
    net, comp, _ = _run(True, iters=5)
    assert comp.store.current_bytes == 0  # every slot consumed exactly once
    # the two max-pools after stored ReLU outputs are MARKER slots (recomputed
    # in backward from the decompressed ReLU output), every iteration
    assert all(r.markers == 2 for r in comp.records)


def test_memory_budget_batch_planner_on_device():
    """with a budget, the compressor recommends a batch from the observed
    ratios once two intervals are planned (training.py:401-416); a budget
    below the stored bytes counts reserve breaches (:420-426)"""
    from paper_2111_09562_b200.hooks import device_memory_budget

    budget = device_memory_budget()
    assert budget > 0
    _, comp, _ = _run(True, iters=7, budget=budget)
    assert comp.controller.intervals_planned >= 2 and comp.batch_size is not None
    assert comp.batch_size >= 16 and comp.reserve_breaches == 0
    # per-sample costs of the three stored activations, measured in the pack hook
    assert set(comp._per_sample) == set(comp.layers)
    tight = comp.fixed_bytes + 1  # fixed bytes alone fill the usable budget
    _, comp2, _ = _run(True, iters=3, budget=int(tight / 0.95) + 1)
    assert comp2.reserve_breaches >= 1


def _train_tv(name, batch, hw, iters, W=2, capture_at=None):
    tv = pytest.importorskip("torchvision")
    torch.manual_seed(0)
    net = getattr(tv.models, name)(num_classes=100).cuda()
    opt = torch.optim.SGD(net.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(net), opt,
                                pb.ControllerConfig(W_default=W, W_floor=1))
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(batch, 3, hw, hw, device="cuda", generator=g)
    y = torch.randint(0, 100, (batch,), device="cuda", generator=g)
    losses = []
    for it in range(iters):
        if capture_at is not None and it == capture_at:
            comp.capture_next_iteration()
        opt.zero_grad()
        with comp.iteration():
            loss = torch.nn.functional.cross_entropy(net(x), y)
            loss.backward()
        opt.step()
        comp.after_step()
        losses.append(float(loss))
        assert len(comp.store) == 0
    return net, comp, losses


def test_resnet50_trains_with_compressed_activations(oracle):
    """torchvision ResNet-50 (Bottleneck blocks share one ReLU module per
    block, residual adds in place): every conv call's ReLU output is a slot,
    compressed at its planned eb from the second interval on; the containers
    the hooks built are the reference's bytes (sampled tensors vs oracle)."""
    net, comp, losses = _train_tv("resnet50", 8, 64, 6, capture_at=4)
    assert all(math.isfinite(v) for v in losses)
    r = comp.records[-1]
    assert len(r.slots) == 49 and comp.plan is not None
    blocks = {s.rsplit(".", 1)[0] for s in r.slots if s.startswith("layer")}
    done = {s.rsplit(".", 1)[0] for s in r.compressed}
    assert len(blocks) == 16 and blocks <= done  # >= 1 compressed slot in every Bottleneck
    assert r.stored_bytes < r.raw_bytes
    assert comp.consumer_names()["layer1.0.conv3"] == "layer1.1.conv1"
    # hooks' containers vs the reference codec on the same tensors
    assert comp.captured
    for slot, (xh, c, eb) in list(comp.captured.items())[::6]:
        ref = oracle.compress(xh, eb, debug=False)
        assert c.to_bytes() == ref.blob, slot
        out, _ = pb.decompress_device(c, dtype=torch.float32)
        want = oracle.decompress_blob(ref.blob, xh.size).astype(np.float32)  # noqa
        assert np.array_equal(out.reshape(-1).cpu().numpy().view(np.uint32), want.view(np.uint32)), slot


def test_vgg16_trains_with_compressed_activations():
    net, comp, losses = _train_tv("vgg16", 4, 64, 5)
    assert all(math.isfinite(v) for v in losses)
    r = comp.records[-1]
    assert len(r.slots) == 13 and r.markers == 5 and len(r.compressed) >= 1
    assert r.stored_bytes < r.raw_bytes and r.device_bytes >= r.stored_bytes  # the decode index is extra


def test_eb_follows_the_current_batch():
    """N in the error model is the current iteration's batch (reference
    training.py:380-390 uses B after choose_batch_size): after the batch
    doubles, the next plan uses N = 32."""
    from paper_2111_09562_b200 import controller as ctl

    net = _net()
    opt = torch.optim.SGD(net.parameters(), lr=0.01, momentum=0.9)
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(net), opt,
                                pb.ControllerConfig(W_default=2, W_floor=1))
    g = torch.Generator(device="cuda").manual_seed(1)
    for it in range(6):
        b = 16 if it < 3 else 32
        x = torch.randn(b, 3, 32, 32, device="cuda", generator=g)
        y = torch.randint(0, 10, (b,), device="cuda", generator=g)
        opt.zero_grad()
        with comp.iteration():
            torch.nn.functional.cross_entropy(net(x), y).backward()
        opt.step()
        comp.after_step()
        if comp.plan is not None and comp.plan.interval_index >= 2:
            break
    assert comp._batch == 32
    for row in comp.plan.detail:
        if not row.skip:
            assert row.eb == ctl.estimate_eb(row.sigma_target, comp.config.a, row.L_bar, 32, row.R)
