"""GPU: training with compressed activations through saved_tensors_hooks."""
import math

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
