"""Benchmark: activation compress+decompress on B200 (contract in the task spec).

Workload (default `alexnet256`, BASELINE.json configs[1]): the five conv/ReLU
activations of torchvision AlexNet at batch 256 on synthetic 224x224 data
(random init), each with the ADAPTIVE error bound the controller derives from
live statistics (R, L_bar, M_avg after two SGD-momentum steps; reference
controller.py:196-232 / errorprop.py:104-124).  One step = compress +
decompress of the whole activation set (124.2 M fp32 elements, 497 MB).

Beside it, in the same line: `c1` (SURVEY config 1, relu-normal
[32,64,56,56] at relative eb 1e-2; the reference's own CPU-runnable case),
and the training legs (configs 2-4: AlexNet b256, VGG-16 b128, ResNet-50
b256 with compressed activations through the hooks vs the same model
uncompressed).  Other workloads: `sweep:<MB>:<rel>` (config 5 cells).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload W]

Rank 0 prints one JSON line.  `value` = whole-job GB/s of fp32 activations
(4n bytes per step) through compress+decompress with inputs resident in HBM;
`e2e` = the same through host buffers (pinned H2D + D2H in the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# deterministic cuBLAS / cuDNN: both arms (separate processes) derive the
# same activations and therefore the same adaptive error bounds
os.environ.setdefault("CUBLAS_WORKSPACE_CONFIG", ":4096:8")

METRIC = "activation compress+decompress GB/s/GPU vs HBM peak; compression ratio; images/s"

KERNEL_NAMES = {"quant": "k1_quant_lorenzo_hist", "codebook": "k2r_codebook (+ k2s_emit)",
                "count": "k3_seg_count (+ CTA-total scan in its last CTA)", "pack": "k3_seg_pack",
                "lut": "k_build_lut(8)", "decode": "k4l_decode (lane per 128-symbol chunk, one-lookup prefix table)"}


def _deterministic():
    import torch

    torch.backends.cudnn.deterministic = True
    torch.backends.cudnn.benchmark = False


def _timeline():
    """(kind name, start ms, end ms) of every launch timed since the last
    call (libactc actc_debug_timeline; consumes the timing records)."""
    import ctypes as C

    from paper_2111_09562_b200 import _lib

    L = _lib.lib()
    L.actc_debug_timeline.argtypes = [C.POINTER(C.c_double), C.c_int]
    L.actc_debug_timeline.restype = C.c_int
    cap = 1 << 16
    buf = (C.c_double * (4 * cap))()
    n = L.actc_debug_timeline(buf, cap)
    kinds = _lib.KERNEL_KINDS
    return [(kinds[int(buf[4 * i])], buf[4 * i + 1], buf[4 * i + 2]) for i in range(n)]


def _union_ms(iv):
    """Length of the union of [a, b) intervals."""
    tot, end = 0.0, None
    for a, b in sorted(iv):
        if end is None or a > end:
            tot += b - a
            end = b
        elif b > end:
            tot += b - end
            end = b
    return tot


def _shares_ms(timeline, kinds):
    """Step time attributed to each kind: every instant is split evenly among
    the kinds (of `kinds`) with a launch running then.  A kind whose
    launches overlap other kinds' (pack beside count and K1) gets less than
    its busy time; one that runs alone (the decoders) keeps all of it."""
    ev = []
    for k, a, b in timeline:
        if k in kinds and b > a:
            ev.append((a, 1, k))
            ev.append((b, -1, k))
    ev.sort(key=lambda e: (e[0], e[1]))
    share = {k: 0.0 for k in kinds}
    live = {}
    prev = None
    for t, d, k in ev:
        if prev is not None and live and t > prev:
            for kk in live:
                share[kk] += (t - prev) / len(live)
        live[k] = live.get(k, 0) + d
        if live[k] == 0:
            del live[k]
        prev = t
    return share


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------


def _host_stats(acts, grads, moms, batch):
    """R, L_bar, M_avg of each layer on the host (the reference arm): the
    reference's own reductions restated by the oracle (tensor.py:171-192,
    training.py:358-361, nn.py:249-253) -- no libactc in that process."""
    from oracle import oracle as orc

    orc.build()
    out = []
    for a, g, v in zip(acts, grads, moms):
        a_h = a.detach().reshape(-1).cpu().numpy()
        g_h = (g * batch).detach().cpu().numpy()
        out.append((orc.count_nonzero(a_h) / a_h.size, orc.lbar(g_h.reshape(g_h.shape[0], -1)),
                    orc.mean_abs(v.detach().reshape(-1).cpu().numpy())))
    return out


def _device_stats(acts, grads, moms, batch):
    """R, L_bar, M_avg on the GPU (K5 reductions, libactc)."""
    from paper_2111_09562_b200 import tensor as pt

    return [(pt.count_nonzero(a) / a.numel(), pt.per_sample_max(g * batch)[1], pt.mean_abs(v))
            for a, g, v in zip(acts, grads, moms)]


def alexnet_activations(batch=256, seed=0, device="cuda", stats="device", keep_stat_inputs=False):
    """Post-ReLU outputs of AlexNet's five convs + adaptive eb per layer.
    stats: "device" (K5 kernels) or "host" (oracle restatement; reference arm)."""
    import torch
    import torchvision

    from paper_2111_09562_b200 import controller as ctl

    _deterministic()
    torch.manual_seed(seed)
    m = torchvision.models.alexnet(num_classes=1000).to(device)
    for mod in m.modules():
        if isinstance(mod, torch.nn.ReLU):
            mod.inplace = False
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    relus = [m.features[i] for i in (1, 4, 7, 9, 11)]
    consumers = [m.features[3], m.features[6], m.features[8], m.features[10], m.classifier[1]]
    acts, grads = {}, {}
    hooks = []
    for i, r in enumerate(relus):
        hooks.append(r.register_forward_hook(lambda mod, inp, out, i=i: acts.__setitem__(i, out.detach())))
    for i, c in enumerate(consumers):
        hooks.append(c.register_full_backward_hook(lambda mod, gi, go, i=i: grads.__setitem__(i, go[0].detach())))
    g = torch.Generator(device=device).manual_seed(seed)
    for _ in range(2):
        x = torch.randn(batch, 3, 224, 224, device=device, generator=g)
        y = torch.randint(0, 1000, (batch,), device=device, generator=g)
        loss = torch.nn.functional.cross_entropy(m(x), y)
        opt.zero_grad(set_to_none=True)
        loss.backward()
        opt.step()
    for h in hooks:
        h.remove()
    layers = [acts[i].contiguous() for i in range(5)]
    gl = [grads[i] for i in range(5)]
    moms = [opt.state[c.weight]["momentum_buffer"] for c in consumers]
    # per-sample (un-averaged) loss gradient: mean-reduced CE scales by 1/B (training.py:303)
    st = (_device_stats if stats == "device" else _host_stats)(layers, gl, moms, batch)
    stats_l = [ctl.LayerTrainingStats(layer_id=f"conv{i + 1}", R=R, L_bar=Lb, M_avg=M, N=batch)
               for i, (R, Lb, M) in enumerate(st)]
    plan = ctl.plan_compression(stats_l, ctl.ControllerConfig(), interval_index=1)
    ebs = [plan.eb[f"conv{i + 1}"] for i in range(5)]
    info = [dict(layer=s.layer_id, shape=list(layers[i].shape), R=s.R, L_bar=s.L_bar, M_avg=s.M_avg, eb=ebs[i])
            for i, s in enumerate(stats_l)]
    stat_inputs = None
    if keep_stat_inputs:
        stat_inputs = [((gg * batch).cpu().numpy(), v.reshape(-1).cpu().numpy()) for gg, v in zip(gl, moms)]
    del m, opt, acts, grads, gl, moms
    torch.cuda.empty_cache()
    return layers, ebs, info, stat_inputs


def relu_normal_tensor(shape, seed, device="cuda"):
    import torch

    g = torch.Generator(device=device).manual_seed(seed)
    return torch.randn(*shape, device=device, generator=g).clamp_min_(0).contiguous()


def build_workload(name, device="cuda", stats="device", keep_stat_inputs=False):
    """Returns (tensors, ebs, info dict, batch, stat_inputs)."""
    import torch

    if name == "alexnet256":
        layers, ebs, info, si = alexnet_activations(256, 0, device, stats, keep_stat_inputs)
        return layers, ebs, {"workload": "alexnet_b256_conv_relu_activations", "layers": info,
                             "eb_mode": "adaptive (controller on live R, L_bar, M_avg after 2 SGD steps)"}, 256, si
    if name == "c1":
        x = np.maximum(np.random.default_rng(0).normal(0, 1, 32 * 64 * 56 * 56), 0).astype(np.float32)
        eb = 1e-2 * float(x.max() - x.min())
        t = torch.from_numpy(x.reshape(32, 64, 56, 56)).to(device)
        return [t], [eb], {"workload": "c1_relu_normal_32x64x56x56", "eb_mode": "rel 1e-2 of range", "eb": eb}, 32, None
    if name.startswith("sweep:"):
        _, mb, rel = name.split(":")
        n = int(float(mb) * (1 << 20)) // 4
        t = relu_normal_tensor((n,), 1234, device)
        eb = float(rel) * float((t.max() - t.min()).item())
        return [t], [eb], {"workload": f"sweep_{mb}MB_rel{rel}", "eb_mode": f"rel {rel} of range", "eb": eb}, 1, None
    raise SystemExit(f"unknown workload {name}")


def line_config(info, world, batch):
    """The `config` object both arms print (identical for the same workload)."""
    cfg = dict(info)
    cfg.update({"parallelism": f"dp{world} (independent shards, no data-path collective)",
                "global_batch": batch * world,
                "l2": "GPU arm: flushed (256 MB memset) between timed steps; reference arm: host"})
    return cfg


# ---------------------------------------------------------------------------
# clocks sampling (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------


class ClockSampler:
    """SM clock + clock-event (throttle) reasons sampled through NVML (the
    library nvidia-smi reads) every 5 ms during the timed region, plus one
    synchronous sample at entry and exit."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()
        self.h = None

    def _sample(self):
        import pynvml

        try:
            sm = pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            self.samples.append((sm, rs))
        except Exception:
            pass

    def _loop(self):
        while not self._stop.wait(0.005):
            self._sample()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.h = None
        return self

    def __exit__(self, *a):
        if self.h is not None:
            self._stop.set()
            self.t.join(timeout=2)
            self._sample()

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": "NVML (nvmlDeviceGetClockInfo / "
                "nvmlDeviceGetCurrentClocksEventReasons), 5 ms period"}


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port: the reference itself is Python and
# does not travel to the GPU box)
# ---------------------------------------------------------------------------


def cpu_roundtrip(tasks, threads, keep=False):
    """Run oracle compress+decompress on (array, eb) tasks with a thread pool
    (ctypes releases the GIL).  Returns (bytes processed, wall seconds,
    [(blob, fp64 reconstruction)] if keep)."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as orc

    orc.build()

    def one(task):
        x, eb = task
        c = orc.compress(x, eb, debug=False)
        rec = orc.decompress_blob(c.blob, x.size)
        return x.nbytes, ((c.blob, rec) if keep else None)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        res = list(ex.map(one, tasks))
    wall = time.perf_counter() - t0
    return sum(r[0] for r in res), wall, [r[1] for r in res]


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_tasks_for(tensors, ebs, max_elems=None):
    tasks = []
    for t, eb in zip(tensors, ebs):
        a = t.detach().cpu().numpy()  # shaped: CMTZ records the dims
        if max_elems:
            a = a.reshape(-1)[:max_elems]
        tasks.append((np.ascontiguousarray(a), float(eb)))
    return tasks


def run_reference(args, rank, world):
    """`--impl reference`: the reference algorithm (oracle port) on host
    cores.  This process never loads libactc: activations come from torch,
    the statistics from the oracle's restatement of the reference's
    reductions, the error bounds from the controller's host arithmetic."""
    import torch

    if rank != 0:
        return None
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    tensors, ebs, info, batch, _ = build_workload(args.workload, dev, stats="host")
    tasks = cpu_tasks_for(tensors, ebs)
    in_bytes = sum(x.nbytes for x, _ in tasks)
    threads = host_threads()
    # every step = the whole workload; all steps' tensors are independent, so
    # they run concurrently across the host threads (per-tensor parallelism)
    for _ in range(args.warmup):
        cpu_roundtrip(tasks[-1:], 1)
    total, wall, _ = cpu_roundtrip(tasks * args.steps, threads)
    gbs = total / wall / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": line_config(info, world, batch),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} x full workload ({in_bytes / 1e6:.1f} MB fp32 per step), "
                                   "oracle/actc_oracle.c (C restatement of actcomp codec.py/huffman.py), "
                                   "one tensor per thread"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs_loaded": _repo_libs_loaded(),
    }
    return line


def _repo_libs_loaded():
    """shared objects from this repo mapped into the process (the reference
    arm must show only oracle/liboracle.so)"""
    try:
        with open("/proc/self/maps") as fh:
            paths = {ln.split()[-1] for ln in fh if ln.rstrip().endswith(".so")}
    except OSError:
        return None
    real = os.path.realpath(ROOT)
    return sorted(os.path.relpath(p, real) for p in paths if os.path.realpath(p).startswith(real))


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------


class CodecTimer:
    """compress_batch + decompress_batch of a tensor set, timed per step on
    the device (CUDA events, L2 flushed between steps)."""

    def __init__(self, tensors, ebs, dev):
        import torch

        import paper_2111_09562_b200 as pb

        self.pb = pb
        self.tensors = tensors
        self.params = [pb.CodecParams(eb=eb) for eb in ebs]
        self.outs = [torch.empty_like(t) for t in tensors]
        self.stream = torch.cuda.current_stream()
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
        self.comp = None

    def ev(self):
        import torch

        return torch.cuda.Event(enable_timing=True)

    def step(self, record=None):
        # compress the whole activation set with one host sync (concurrent
        # codebooks), then decompress the set concurrently (one stream each)
        e0, e1, e2 = self.ev(), self.ev(), self.ev()
        e0.record(self.stream)
        comp = self.pb.compress_batch(self.tensors, self.params)
        e1.record(self.stream)
        self.pb.decompress_batch([c for c, _ in comp], self.outs)
        e2.record(self.stream)
        if record is not None:
            record.append((e0, e1, e2))
        self.comp = comp
        return comp

    def bound_gate(self):
        """device reconstruction must honour the bound: fp32 output =
        fp32(reference fp64 recon), tolerance eb + ulp(x_hat)/2"""
        import torch

        torch.cuda.synchronize()
        self.pb.check_decode_status()
        for t, o, p in zip(self.tensors, self.outs, self.params):
            eb = p.eb
            half_ulp = (torch.nextafter(o.abs(), torch.full_like(o, float("inf"))) - o.abs()).double() / 2
            err = (t.double() - o.double()).abs()
            ok = (err <= eb + half_ulp) | ((o == 0) & (t.abs().double() <= 2 * eb))
            assert bool(ok.all()), f"bound violated: {int((~ok).sum())} elements"
            del half_ulp, err, ok
        torch.cuda.empty_cache()

    def timed(self, steps):
        """per-step ms, phase ms (summed), from CUDA events on the caller stream"""
        import torch

        step_ms, phase = [], {"compress": 0.0, "decompress": 0.0}
        for _ in range(steps):
            self.flush.zero_()
            s0, s1 = self.ev(), self.ev()
            s0.record(self.stream)
            rec = []
            self.step(rec)
            s1.record(self.stream)
            s1.synchronize()
            step_ms.append(s0.elapsed_time(s1))
            e0, e1, e2 = rec[0]
            phase["compress"] += e0.elapsed_time(e1)
            phase["decompress"] += e1.elapsed_time(e2)
        torch.cuda.synchronize()
        return step_ms, phase


def _max_over_ranks(v, world, dev):
    if world == 1:
        return v
    import torch

    t = torch.tensor([v], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_c1(args, dev, world):
    """BASELINE configs[0] / SURVEY C1 beside the headline: GB/s, ratio and
    round-trip roofline fraction of the relu-normal [32,64,56,56] tensor at
    relative eb 1e-2 (reference ratio 6.982)."""
    import torch

    tensors, ebs, info, _, _ = build_workload("c1", dev)
    ct = CodecTimer(tensors, ebs, dev)
    for _ in range(max(3, args.warmup)):
        ct.step()
    ct.bound_gate()
    # the gate releases the allocator's cache: settle the step's allocations
    # again before the timed region (as the headline leg does)
    for _ in range(2):
        ct.step()
    torch.cuda.synchronize()
    steps = max(args.steps, 20)
    step_ms, phase = ct.timed(steps)
    ms = _max_over_ranks(sum(step_ms), world, dev) / steps
    n = tensors[0].numel()
    C = ct.comp[0][1].compressed_bytes
    peak, _ = _peaks()
    return {"workload": info["workload"], "eb": ebs[0], "value": world * 4 * n / (ms * 1e-3) / 1e9, "unit": "GB/s",
            "ms_per_step": ms, "compression_ratio": ct.comp[0][1].ratio, "compressed_bytes": C,
            "roofline_fraction_round_trip": (8 * n + 2 * C) / (ms * 1e-3) / 1e9 / peak,
            "phase_ms_per_step": {k: v / steps for k, v in phase.items()}, "steps": steps,
            "step_ms_min_median_max": [min(step_ms), sorted(step_ms)[steps // 2], max(step_ms)],
            "_tensors": tensors, "_ebs": ebs, "_comp": ct.comp, "_outs": ct.outs}


def parity_block(tensors, ebs, comp, outs, threads):
    """Bit-exact parity of what was benchmarked: every layer's CMTZ blob vs
    the oracle's, and the fp32 reconstruction vs fp32(oracle fp64)."""
    tasks = cpu_tasks_for(tensors, ebs)
    nbytes, wall, res = cpu_roundtrip(tasks, threads, keep=True)
    blobs_equal = recon_equal = 0
    ratios_equal = 0
    for (c, rep), o, (blob, rec) in zip(comp, outs, res):
        blobs_equal += int(c.to_bytes() == blob)
        ratios_equal += int(rep.ratio == (4 * o.numel()) / len(blob))
        got = o.detach().reshape(-1).cpu().numpy().view(np.uint32)
        recon_equal += int(np.array_equal(got, rec.astype(np.float32).view(np.uint32)))
    return {"blobs_equal": blobs_equal, "recon_equal": recon_equal, "ratios_equal": ratios_equal,
            "of": len(comp)}, nbytes, wall


def run_gpu(args, rank, world):
    import torch

    import paper_2111_09562_b200 as pb  # noqa: F401
    from paper_2111_09562_b200 import _lib

    dev = torch.device("cuda", torch.cuda.current_device())
    want_cpu = world == 1 and not args.no_cpu
    tensors, ebs, info, batch, stat_inputs = build_workload(args.workload, dev, keep_stat_inputs=want_cpu)
    n_total = sum(t.numel() for t in tensors)
    in_bytes = 4 * n_total
    ct = CodecTimer(tensors, ebs, dev)
    for _ in range(args.warmup):
        ct.step()
    ct.bound_gate()
    for _ in range(2):
        ct.step()
    torch.cuda.synchronize()

    # timed region: per-step events, L2 flushed between steps (untimed)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    _lib.kernel_stats()  # reset the per-kind launch counters
    with ClockSampler(dev.index if os.environ.get("CUDA_VISIBLE_DEVICES") is None else 0) as clk:
        step_ms, phase = ct.timed(args.steps)
    launch_stats = _lib.kernel_stats()  # launches counted inside the timed region
    comp = ct.comp
    ratios = [r.ratio for _, r in comp]
    C = sum(r.compressed_bytes for _, r in comp)
    dev_bytes = sum(c.device_nbytes for c, _ in comp)
    # kernel breakdown: the same K steps again with every library launch
    # bracketed by CUDA events on its own stream (kept out of the headline
    # region: the event records cost host time between launches)
    _lib.timing_enable(True)
    for _ in range(args.steps):
        ct.flush.zero_()
        ct.step()
    torch.cuda.synchronize()
    _lib.timing_enable(False)
    timeline = _timeline()
    kstats = _lib.kernel_stats()
    total_ms = _max_over_ranks(sum(step_ms), world, dev)
    ms_per_step = total_ms / args.steps
    gbs = world * in_bytes * args.steps / (total_ms * 1e-3) / 1e9

    # roofline of the dominant kernel: algorithmic bytes per step per kind
    # as stated in DESIGN.md section 4 (index = 16 B per 128-symbol chunk)
    sb = 2  # u16 symbols (radius <= 2^15)
    nidx = sum((t.numel() + 127) // 128 for t in tensors)
    alg_step = {
        "quant": 4 * n_total + sb * n_total + 8 * nidx,  # read fp32, write symbols + chunk lattice
        "count": sb * n_total,  # read symbols
        "pack": sb * n_total + C + 8 * nidx,  # read symbols, write bitstream + outliers + chunk offsets
        "decode": C + 16 * nidx + 4 * n_total,  # read bitstream + chunk index, write fp32
    }
    kernels = {}
    for kind, (nl, _) in kstats.items():
        if nl == 0:
            continue
        iv = [(a, b) for k, a, b in timeline if k == kind]
        ms = sum(b - a for a, b in iv)
        busy = _union_ms(iv)
        ent = {"launches_per_step": nl / args.steps, "ms_per_step": ms / args.steps,
               "busy_ms_per_step": busy / args.steps}
        if kind in alg_step and busy > 0:
            ent["alg_bytes_per_launch"] = alg_step[kind] * args.steps / nl
            # the tensors' launches of one kind overlap on their streams: the
            # kind's throughput is its bytes over the time any launch of it runs
            ent["achieved_gbs"] = alg_step[kind] * args.steps / (busy * 1e-3) / 1e9
            ent["achieved_gbs_per_launch_avg"] = alg_step[kind] * args.steps / (ms * 1e-3) / 1e9
        kernels[kind] = ent
    hbm_kinds = [k for k in ("quant", "count", "pack", "decode") if k in kernels]
    # dominant = the largest share of the step (each instant split among the
    # bandwidth kernels running then); busy time alone flips between pack and
    # the decoders from run to run (pack's launches overlap count's and K1's)
    shares = _shares_ms(timeline, set(hbm_kinds))
    for k in hbm_kinds:
        kernels[k]["step_share_ms_per_step"] = shares[k] / args.steps
    dom = max(hbm_kinds or list(kernels), key=lambda k: kernels[k].get("step_share_ms_per_step",
                                                                       kernels[k]["busy_ms_per_step"]))
    peak, peak_kind = _peaks()
    achieved = kernels[dom].get("achieved_gbs", 0.0)
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            traffic = json.load(fh).get(args.workload, {}).get(dom)
    except Exception:
        pass
    gpu_launches = sum(nl for nl, _ in launch_stats.values())

    e2e_gbs = run_e2e(args, ct, world, dev, in_bytes)

    line = None
    if rank == 0:
        ratio_total = in_bytes / C
        line = {
            "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (AlexNet random init, randn images)"
            if args.workload == "alexnet256" else "synthetic", "config": line_config(info, world, batch),
            "compression_ratio": ratio_total, "per_layer_ratio": ratios,
            "bytes_in_per_step_per_gpu": in_bytes, "compressed_bytes_per_step_per_gpu": C,
            "device_bytes_of_containers": dev_bytes,
            "phase_ms_per_step": {k: v / args.steps for k, v in phase.items()},
            "codec_images_per_s": world * batch / (ms_per_step * 1e-3),
            "roofline_fraction_round_trip": (world * (8 * n_total + 2 * C) / (ms_per_step * 1e-3) / 1e9) / peak,
            "roofline": {"bound": "hbm", "kernel": KERNEL_NAMES.get(dom, dom), "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_launch": kernels[dom].get("alg_bytes_per_launch"),
                         "avg_launch_ms": kernels[dom]["ms_per_step"] / kernels[dom]["launches_per_step"],
                         "busy_ms_per_step": kernels[dom]["busy_ms_per_step"],
                         "achieved_per_launch_avg": kernels[dom].get("achieved_gbs_per_launch_avg"),
                         "frac_per_launch_avg": (kernels[dom].get("achieved_gbs_per_launch_avg") or 0.0) / peak,
                         "step_share_ms_per_step": kernels[dom].get("step_share_ms_per_step"),
                         "timing": "CUDA events around every launch on its own stream, a second pass of the "
                                   "same K steps; achieved = the kernel's algorithmic bytes per step / the time "
                                   "per step during which at least one of its launches runs (the tensors' "
                                   "launches overlap on their streams); the per-launch-average figure "
                                   "(bytes per launch / mean launch duration) is beside it; dominant = the "
                                   "bandwidth kernel with the largest share of the step (each instant split "
                                   "evenly among the bandwidth kernels running then)"},
            "kernels": kernels,
            "e2e": {"value": e2e_gbs, "unit": "GB/s", "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": in_bytes},
            "gpu_launches": gpu_launches,  # counted by libactc (actc_kernel_stats) over the timed region
            "clocks": clk.summary(),
        }
    c1 = None
    if args.workload == "alexnet256" and not args.no_c1:
        c1 = run_c1(args, dev, world)
    if line is not None and want_cpu:
        threads = min(host_threads(), len(tensors))
        par, nbytes, wall = parity_block(tensors, ebs, comp, ct.outs, threads)
        line["cpu_baseline"] = {"value": nbytes / wall / 1e9, "unit": "GB/s", "cores": threads, "kind": "port",
                                "sample": f"one full step ({nbytes / 1e6:.1f} MB fp32) through oracle/actc_oracle.c, "
                                          "one tensor per thread"}
        if stat_inputs is not None:
            # the K5 statistics that set the benchmarked error bounds vs the
            # oracle's restatement of the reference reductions
            from oracle import oracle as orc

            eq = 0
            for lay, (g, v), t in zip(info["layers"], stat_inputs, tensors):
                a = t.reshape(-1).cpu().numpy()
                eq += int(lay["R"] == orc.count_nonzero(a) / a.size and
                          lay["L_bar"] == orc.lbar(g.reshape(g.shape[0], -1)) and lay["M_avg"] == orc.mean_abs(v))
            par["stats_equal"] = eq
        line["parity"] = par
    if line is not None and c1 is not None:
        if want_cpu:
            p1, _, _ = parity_block(c1["_tensors"], c1["_ebs"], c1["_comp"], c1["_outs"], 1)
            c1["parity"] = p1
        line["c1"] = {k: v for k, v in c1.items() if not k.startswith("_")}
    return line


def run_e2e(args, ct, world, dev, in_bytes):
    """end to end through host buffers (pinned H2D of inputs, D2H of
    outputs), the public API, per-tensor pipeline"""
    import torch

    pb = ct.pb
    tensors, params, outs, stream = ct.tensors, ct.params, ct.outs, ct.stream
    host_in = [t.cpu().pin_memory() for t in tensors]
    host_out = [torch.empty(t.shape, dtype=torch.float32).pin_memory() for t in tensors]
    dev_in = [torch.empty_like(t) for t in tensors]
    h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
    order = sorted(range(len(tensors)), key=lambda i: -tensors[i].numel())

    def e2e_step():
        # all host->device copies are queued up front (largest first); each
        # tensor is compressed as soon as its copy lands, reconstructed, and
        # copied back while later tensors are still crossing PCIe
        cur = torch.cuda.current_stream()
        h2d_s.wait_stream(cur)
        ready = {}
        for i in order:
            with torch.cuda.stream(h2d_s):
                dev_in[i].copy_(host_in[i], non_blocking=True)
            ready[i] = h2d_s.record_event()
        for i in order:
            (c, _), = pb.compress_batch([dev_in[i]], [params[i]], ready=[ready[i]])
            done = []
            pb.decompress_batch([c], [outs[i]], done=done)
            d2h_s.wait_event(done[0])
            with torch.cuda.stream(d2h_s):
                host_out[i].copy_(outs[i], non_blocking=True)
        cur.wait_stream(d2h_s)

    # the pipeline runs on its own (non-default) stream: work on the legacy
    # default stream would serialise with the copy streams
    e2e_main = torch.cuda.Stream()
    for _ in range(max(1, args.warmup // 2)):
        e2e_main.wait_stream(stream)
        with torch.cuda.stream(e2e_main):
            e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e2e_ms = 0.0
    for _ in range(args.steps):
        ct.flush.zero_()
        e2e_main.wait_stream(stream)
        s0, s1 = ct.ev(), ct.ev()
        with torch.cuda.stream(e2e_main):
            s0.record(e2e_main)
            e2e_step()
            s1.record(e2e_main)
        s1.synchronize()
        e2e_ms += s0.elapsed_time(s1)
    e2e_ms = _max_over_ranks(e2e_ms, world, dev)
    del host_in, host_out, dev_in
    return world * in_bytes * args.steps / (e2e_ms * 1e-3) / 1e9


# ---------------------------------------------------------------------------
# training legs (configs 2-4)
# ---------------------------------------------------------------------------

TRAIN_LEGS = {"alexnet": 256, "vgg16": 128, "resnet50": 256}


def run_training(model_name, batch, world, iters=6, warm=4, spot_check=False):
    """Training with compressed activations (hooks, adaptive eb) vs the same
    run uncompressed: images/s, peak memory, per-layer ratio/eb; with
    spot_check, one stored tensor per layer compressed inside the hooks is
    checked against the oracle (blob + reconstruction).  The warm-up runs
    W = 2 intervals (plans from live statistics); the timed iterations are
    steady-state compressed iterations (the reference's W_default = 1000
    puts one statistics collection per 1000 iterations)."""
    import torch
    import torchvision

    import paper_2111_09562_b200 as pb
    from paper_2111_09562_b200 import _lib
    from paper_2111_09562_b200.hooks import ActivationCompressor

    dev = torch.device("cuda", torch.cuda.current_device())
    rank = torch.distributed.get_rank() if world > 1 else 0
    _lib.release_contexts()  # the codec legs' scratch is not the training's
    out = {}
    for mode in ("baseline", "compressed"):
        torch.manual_seed(0)
        m = getattr(torchvision.models, model_name)(num_classes=1000).to(dev)
        opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
        ddp = m
        if world > 1:
            ddp = torch.nn.parallel.DistributedDataParallel(m, device_ids=[dev.index])
        comp = None
        if mode == "compressed":
            comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt,
                                        pb.ControllerConfig(W_default=2, W_floor=1))
        g = torch.Generator(device=dev).manual_seed(rank)
        x = torch.randn(batch, 3, 224, 224, device=dev, generator=g)
        y = torch.randint(0, 1000, (batch,), device=dev, generator=g)

        def it():
            opt.zero_grad(set_to_none=True)
            if comp:
                with comp.iteration():
                    torch.nn.functional.cross_entropy(ddp(x), y).backward()
            else:
                torch.nn.functional.cross_entropy(ddp(x), y).backward()
            opt.step()
            if comp:
                comp.after_step()

        for _ in range(warm):
            it()
        if comp:
            comp.next_collection = comp.it + 1000
            # two iterations at the final plan before timing: its first
            # iteration sizes the caps for the new error bounds
            it()
            it()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats(dev)
        if world > 1:
            torch.distributed.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
        from paper_2111_09562_b200 import codec as _codec
        redos0 = len(_codec.REDOS)
        st0 = torch.cuda.memory_stats(dev)
        evs[0].record()
        for i in range(iters):
            it()
            evs[i + 1].record()
        evs[-1].synchronize()
        ms = _max_over_ranks(evs[0].elapsed_time(evs[-1]), world, dev)
        rec = {"images_per_s": world * batch * iters / (ms * 1e-3), "ms_per_iter": ms / iters,
               "ms_each_iter": [round(evs[i].elapsed_time(evs[i + 1]), 2) for i in range(iters)],
               "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9}
        st1 = torch.cuda.memory_stats(dev)
        # allocator events inside the timed window (each cudaMalloc / retry
        # synchronises the device): evidence for an outlier iteration
        rec["allocator_in_timed_window"] = {
            "cuda_mallocs": st1.get("num_device_alloc", 0) - st0.get("num_device_alloc", 0),
            "alloc_retries": st1.get("num_alloc_retries", 0) - st0.get("num_alloc_retries", 0)}
        if comp:
            rec["recompressions_in_timed_window"] = len(_codec.REDOS) - redos0
        if comp:
            # the codec contexts' scratch is cudaMalloc'ed by the library,
            # outside torch's allocator: reported beside the allocator peak
            sb = _lib.scratch_bytes(slots=range(comp.batch_flush + 2))
            rec["codec_scratch_gb"] = sb / 1e9
            rec["peak_mem_gb_incl_codec_scratch"] = rec["peak_mem_gb"] + sb / 1e9
            last = [r for r in comp.records if r.compressed][-1:]
            if last:
                r = last[0]
                rec["activation_bytes_raw"] = r.raw_bytes
                rec["activation_bytes_stored_cmtz"] = r.stored_bytes
                rec["activation_bytes_stored_device"] = r.device_bytes
                rec["stored_slots"] = len(r.slots)
                rec["compressed_slots"] = len(r.compressed)
                rec["markers"] = r.markers
                rec["per_layer"] = {k: {"ratio": v[0], "eb": v[1]} for k, v in r.compressed.items()}
            rec["W"] = comp.controller.W
            if spot_check and rank == 0:
                rec["oracle_spot_check"] = _spot_check(comp, it)
            comp.remove()
        out[mode] = rec
        del m, opt, ddp, comp, x, y
        torch.cuda.empty_cache()
    out["overhead_pct"] = 100.0 * (out["baseline"]["images_per_s"] / out["compressed"]["images_per_s"] - 1.0)
    out["config"] = {"model": model_name, "batch_per_gpu": batch, "image": "224x224 synthetic",
                     "W": "2 in warm-up (plans from live statistics), no collection in the timed window",
                     "optimizer": "SGD momentum 0.9"}
    return out


def run_planner_leg(world, budget_bytes, batch=256, iters=6):
    """The memory-budget batch planner applied (reference training.py:401-416,
    PAPER.md:727): AlexNet with compressed activations under a device memory
    budget equal to the uncompressed b256 run's peak; after two planned
    intervals the compressor's recommended batch (choose_batch_size over the
    observed per-layer ratios) is adopted and trained at -- images/s at that
    batch vs the uncompressed run at b256 (the largest power-of-two batch the
    same budget admits uncompressed)."""
    import torch
    import torchvision

    import paper_2111_09562_b200 as pb
    from paper_2111_09562_b200 import _lib
    from paper_2111_09562_b200.hooks import ActivationCompressor

    dev = torch.device("cuda", torch.cuda.current_device())
    rank = torch.distributed.get_rank() if world > 1 else 0
    _lib.release_contexts()
    torch.manual_seed(0)
    m = torchvision.models.alexnet(num_classes=1000).to(dev)
    opt = torch.optim.SGD(m.parameters(), lr=0.01, momentum=0.9)
    ddp = torch.nn.parallel.DistributedDataParallel(m, device_ids=[dev.index]) if world > 1 else m
    comp = ActivationCompressor(ActivationCompressor.conv_layer_map(m), opt,
                                pb.ControllerConfig(W_default=2, W_floor=1, memory_budget_bytes=int(budget_bytes)),
                                input_sample_bytes=3 * 224 * 224 * 4)
    g = torch.Generator(device=dev).manual_seed(rank)

    def batch_of(b):
        return (torch.randn(b, 3, 224, 224, device=dev, generator=g),
                torch.randint(0, 1000, (b,), device=dev, generator=g))

    def it(x, y):
        opt.zero_grad(set_to_none=True)
        with comp.iteration():
            torch.nn.functional.cross_entropy(ddp(x), y).backward()
        opt.step()
        comp.after_step()

    x, y = batch_of(batch)
    while comp.batch_size is None and comp.it < 12:
        it(x, y)
    b2 = comp.batch_size or batch
    x, y = batch_of(b2)
    for _ in range(2):
        it(x, y)
    comp.next_collection = comp.it + 1000
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        it(x, y)
    e1.record()
    e1.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1), world, dev)
    out = {"budget_gb": budget_bytes / 1e9, "planned_batch": b2, "start_batch": batch,
           "images_per_s": world * b2 * iters / (ms * 1e-3), "ms_per_iter": ms / iters,
           "peak_mem_gb": torch.cuda.max_memory_allocated(dev) / 1e9,
           "reserve_breaches": comp.reserve_breaches,
           "note": "planner model = stored activations (raw bytes / observed ratio) + input + weights and "
                   "velocity (training.py:401-416); peak_mem_gb is the allocator's actual peak at that batch"}
    comp.remove()
    del m, opt, ddp, comp, x, y
    torch.cuda.empty_cache()
    return out


def _spot_check(comp, it, max_slots=8):
    """One more iteration capturing stored activations: each sampled slot's
    container (compressed inside the hooks at the controller's eb) vs the
    oracle on the same tensor -- CMTZ blob, ratio, reconstruction."""
    import torch

    from paper_2111_09562_b200 import decompress_device

    slots = [s for s in comp.records[-1].compressed]
    pick = slots if len(slots) <= max_slots else [slots[int(i * (len(slots) - 1) / (max_slots - 1))]
                                                  for i in range(max_slots)]
    comp.capture_next_iteration(pick)
    it()
    torch.cuda.synchronize()
    tasks = [(x, eb) for x, _, eb in comp.captured.values()]
    _, _, res = cpu_roundtrip(tasks, min(host_threads(), max(1, len(tasks))), keep=True)
    rep = {"slots": list(comp.captured), "blobs_equal": 0, "recon_equal": 0, "of": len(tasks)}
    for (x, c, eb), (blob, rec) in zip(comp.captured.values(), res):
        rep["blobs_equal"] += int(c.to_bytes() == blob)
        o, _ = decompress_device(c, dtype=torch.float32)
        rep["recon_equal"] += int(np.array_equal(o.reshape(-1).cpu().numpy().view(np.uint32),
                                                 rec.astype(np.float32).view(np.uint32)))
    comp.captured = {}
    return rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="alexnet256")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline / parity legs")
    ap.add_argument("--no-train", action="store_true", help="skip the training legs")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 sub-line")
    ap.add_argument("--train", default="alexnet,vgg16,resnet50", help="training legs to run")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    try:
        if args.impl == "reference":
            line = run_reference(args, rank, world)
        else:
            line = run_gpu(args, rank, world)
            if not args.no_train and args.workload == "alexnet256":
                legs = {}
                for name in [s for s in args.train.split(",") if s]:
                    legs[name] = run_training(name, TRAIN_LEGS[name], world, spot_check=not args.no_cpu)
                if "alexnet" in legs:
                    base = legs["alexnet"]["baseline"]
                    pl = run_planner_leg(world, base["peak_mem_gb"] * 1e9)
                    pl["speedup_vs_uncompressed_b256"] = pl["images_per_s"] / base["images_per_s"]
                    legs["alexnet_planner"] = pl
                if line is not None:
                    line["training"] = legs
                    if "alexnet" in legs:
                        line["train_images_per_s"] = legs["alexnet"]["compressed"]["images_per_s"]
        if rank == 0 and line is not None:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
