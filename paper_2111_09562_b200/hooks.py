"""Per-layer activation compression hooks for PyTorch training.

Mirrors the reference's hook API and storage policy
(/root/reference/pkg/src/actcomp/training.py):

* `ActivationStore` -- per-layer slots RAW / COMPRESSED / MARKER with byte
  accounting, put-once / pop-once (LifecycleError), training.py:105-138.
* `ActivationCompressor` -- the train() hook sites (training.py:259-299
  compress after forward, :335-353 lazy decompress in backward, :351-361
  statistics, :381-418 interval boundary) re-expressed for autograd:
  `torch.autograd.graph.saved_tensors_hooks` pack/unpack.  What autograd
  saves for a conv layer is its (post-ReLU) output, which the next layer's
  backward consumes; pack hands it to the GPU codec at the layer's current
  error bound, unpack reconstructs it (fp32, on device).

Policy, as in the reference:
* no compression during the first interval (W iterations) -- there is no
  plan yet (training.py:265-266);
* every W iterations the collection iteration measures R (nonzero ratio of
  the stored, i.e. decompressed, activation), L_bar (per-sample max of the
  loss gradient at the consumer's output, un-averaged) and M_avg (mean |v|
  of the consumer's momentum) and asks the controller for the next plan;
* layers whose eb is None (skip set) stay raw.

Packing is asynchronous: a stored activation's compression is launched on a
side stream as soon as its producer has run (`compress_begin`, no host
sync); the oldest in-flight compression is finished (`compress_end`: plan
read, exact-size container, original released) once more than `batch_flush`
are in flight, so the raw activations of at most that many layers coexist
with their compressed copies.
Under data parallelism the statistics are averaged across ranks before
planning, so every rank compresses with identical error bounds.
"""
from __future__ import annotations

import contextlib
import weakref
from dataclasses import dataclass, field

from . import _lib
from .codec import DEFAULT_RADIUS, CodecParams, compress_begin, compress_end, decompress_device
from .controller import AdaptiveController, ControllerConfig, LayerTrainingStats, choose_batch_size
from .errors import LifecycleError, ParameterError


class ActivationStore:
    """Per-layer slots (reference training.py:105-138)."""

    RAW = "raw"
    COMPRESSED = "compressed"
    MARKER = "marker"

    def __init__(self):
        self._slots: dict[str, tuple[str, object, int]] = {}
        self.current_bytes = 0
        self.peak_bytes = 0

    def put(self, layer_id: str, kind: str, payload, nbytes: int):
        if layer_id in self._slots:
            raise LifecycleError(f"slot {layer_id!r} already filled")
        self._slots[layer_id] = (kind, payload, nbytes)
        self.current_bytes += nbytes
        self.peak_bytes = max(self.peak_bytes, self.current_bytes)

    def pop(self, layer_id: str):
        entry = self._slots.pop(layer_id, None)
        if entry is None:
            raise LifecycleError(f"slot {layer_id!r} missing or already consumed")
        self.current_bytes -= entry[2]
        return entry

    def clear(self):
        self._slots.clear()
        self.current_bytes = 0

    def __contains__(self, layer_id: str) -> bool:
        return layer_id in self._slots


def _key(t):
    return (t.data_ptr(), t._version, tuple(t.shape), tuple(t.stride()))


class _Marker:
    """A cheap layer's saved output (pooling after a stored activation):
    nothing is kept; unpack recomputes it from the stored predecessor
    (reference MARKER slots, training.py:295-296, recompute_cheap :344-347)."""

    __slots__ = ("slot", "mod", "src", "packs", "unpacks", "out", "ref")

    def __init__(self, slot, mod, src, t):
        self.slot = slot
        self.mod = mod
        self.src = src
        self.packs = 1
        self.unpacks = 0
        self.out = None
        self.ref = weakref.ref(t)


class _Handle:
    """One saved fp32 tensor.  Autograd saves a module's output while the op
    runs, before the module's forward hook names it, so every saved tensor
    gets a handle; the producer's forward hook then promotes the handle of
    its output to a stored activation (layer set): raw until the pending
    queue is flushed, compressed after.  Handles nobody promotes pass the
    tensor through."""

    __slots__ = ("layer", "eb", "raw", "comp", "report", "packs", "unpacks", "out", "shape", "ref", "job")

    def __init__(self, t, layer, eb):
        self.layer = layer
        self.eb = eb
        self.raw = t
        self.comp = None
        self.report = None
        self.packs = 1
        self.unpacks = 0
        self.out = None
        self.shape = tuple(t.shape)
        self.job = None  # compress_begin batch while the compression is in flight
        # the tensor's identity: a key (pointer, version, shape, stride) is
        # only unique while the tensor lives -- freed memory is reused
        self.ref = weakref.ref(t)


@dataclass
class IterationRecord:
    iteration: int
    compressed: dict = field(default_factory=dict)  # layer -> (ratio, eb)
    stored_bytes: int = 0
    raw_bytes: int = 0
    markers: int = 0  # cheap-layer outputs recomputed instead of stored


class _LayerMap(dict):
    """conv_layer_map's result: the layer map plus the model it came from
    (whose in-place ReLUs run out of place in collection iterations)."""

    def __init__(self, d, model):
        super().__init__(d)
        self.model = model


class ActivationCompressor:
    """Adaptive activation compression for a PyTorch model.

    layers: {layer_id: (producer_module, consumer_module)} -- the producer's
    forward output is the stored activation (e.g. the ReLU after a conv), the
    consumer is the next parameterised layer whose momentum and output
    gradient set the error bound.  `conv_layer_map` builds this map
    for conv nets (conv -> relu -> ... -> next conv/linear).
    """

    def __init__(self, layers, optimizer, config: ControllerConfig | None = None, radius: int = DEFAULT_RADIUS,
                 preserve_zeros: bool = True, grad_scale=None, batch_flush: int = 1, dist_group=None,
                 sync_stats: bool = True, input_sample_bytes: float | None = None, fixed_bytes: float | None = None,
                 recompute_cheap: bool = True):
        self.layers = dict(layers)
        self._model = getattr(layers, "model", None)
        self.optimizer = optimizer
        self.config = config or ControllerConfig()
        self.controller = AdaptiveController(self.config)
        self.radius = radius
        self.preserve_zeros = preserve_zeros
        self.grad_scale = grad_scale  # None: use the batch size (mean-reduced loss)
        self.batch_flush = batch_flush
        self.dist_group = dist_group
        self.sync_stats = sync_stats
        self.plan = None
        self.it = 0
        self.next_collection = self.controller.W
        self.store = ActivationStore()
        self.records: list[IterationRecord] = []
        self._act_layer: dict = {}
        self._handles: dict = {}
        self._pending: list[_Handle] = []  # compressions launched, not yet synchronised (oldest first)
        self._slot = 0
        self._collecting = False
        self._R: dict[str, float] = {}
        self._bits: dict[str, int] = {}
        self._lbar: dict[str, float] = {}
        self._batch = None
        self._rec = None
        self._hooks = []
        self._bwd_hooks = []
        # memory-budget batch planner (reference training.py:401-426): per-
        # sample bytes of each stored activation, the ratios observed in the
        # current interval, the model's fixed bytes (weights + velocity)
        self.input_sample_bytes = input_sample_bytes
        if fixed_bytes is None:
            fixed_bytes = 2.0 * sum(p.numel() * p.element_size()
                                    for g in optimizer.param_groups for p in g["params"])
        self.fixed_bytes = float(fixed_bytes)
        self.batch_size = None  # recommended batch (choose_batch_size), once planned
        self._per_sample: dict[str, float] = {}
        self._interval_ratios: dict[str, list] = {lid: [] for lid in self.layers}
        for lid, (prod, cons) in self.layers.items():
            self._hooks.append(prod.register_forward_hook(self._fwd_hook(lid)))
        # cheap layers (pooling) fed by a stored activation: their saved
        # outputs become MARKER slots, recomputed in backward
        self._cheap: dict = {}
        self._markers: dict = {}
        if recompute_cheap and self._model is not None:
            import torch.nn as nn

            for name, m in self._model.named_modules():
                if isinstance(m, (nn.MaxPool2d, nn.AvgPool2d)):
                    self._hooks.append(m.register_forward_hook(self._cheap_hook(name)))

    # ---- construction helpers -------------------------------------------
    @staticmethod
    def conv_layer_map(model):
        """{name: (activation module, consumer module)} for every Conv2d: the
        activation is the first ReLU after it (else the conv itself), the
        consumer the next Conv2d / Linear in module registration order
        (reference _consumer_map, training.py:154-166)."""
        import torch.nn as nn

        mods = [(n, m) for n, m in model.named_modules() if not list(m.children())]
        out = {}
        for i, (name, m) in enumerate(mods):
            if not isinstance(m, nn.Conv2d):
                continue
            act, cons = m, None
            for n2, m2 in mods[i + 1:]:
                if isinstance(m2, nn.ReLU) and act is m:
                    act = m2
                if isinstance(m2, (nn.Conv2d, nn.Linear)):
                    cons = m2
                    break
            if cons is not None:
                out[name] = (act, cons)
        return _LayerMap(out, model)

    def _modules(self):
        seen = []
        for prod, cons in self.layers.values():
            for m in (prod, cons):
                if all(m is not x for x in seen):
                    seen.append(m)
        return seen

    def remove(self):
        for h in self._hooks + self._bwd_hooks:
            h.remove()
        self._hooks.clear()
        self._bwd_hooks.clear()

    # ---- hooks ---------------------------------------------------------------
    def _fwd_hook(self, lid):
        def hook(mod, inp, out):
            if self._batch is None and inp and hasattr(inp[0], "shape"):
                self._batch = int(inp[0].shape[0])
            if not hasattr(out, "data_ptr"):
                return
            k = _key(out)
            self._act_layer[k] = (lid, weakref.ref(out))
            h = self._live(self._handles, k)
            if h is not None and h.layer is None:
                self._promote(h, lid)  # saved by the op itself, before this hook
        return hook

    def _cheap_hook(self, name):
        def hook(mod, inp, out):
            if inp and hasattr(inp[0], "data_ptr") and hasattr(out, "data_ptr"):
                src = self._live(self._handles, _key(inp[0]))
                if src is not None and src.layer is not None:
                    self._cheap[_key(out)] = (name, mod, src, weakref.ref(out))
        return hook

    @staticmethod
    def _live(table, k):
        """table[k] if the tensor it was registered for is still alive."""
        e = table.get(k)
        if e is None:
            return None
        ref = e[-1] if isinstance(e, tuple) else e.ref
        if ref() is None:
            del table[k]
            return None
        return e

    def _bwd_hook(self, lid):
        def hook(mod, gin, gout):
            if self._collecting and gout and gout[0] is not None:
                from .tensor import per_sample_max

                scale = self.grad_scale if self.grad_scale is not None else (self._batch or 1)
                _, lbar = per_sample_max(gout[0].detach().float())
                self._lbar[lid] = lbar * scale
        return hook

    def _pack(self, t):
        import torch

        if not (t.is_cuda and t.dtype == torch.float32) or isinstance(t, torch.nn.Parameter):
            return ("raw", t)
        k = _key(t)
        h = self._live(self._handles, k)
        if h is not None:
            h.packs += 1
            return h
        m = self._live(self._markers, k)
        if m is not None:
            m.packs += 1
            return m
        cheap = self._live(self._cheap, k)
        if cheap is not None and cheap[2].ref() is not None:
            src = cheap[2]
            m = _Marker(f"{cheap[0]}@{src.layer}", cheap[1], src, t)
            src.packs += 1  # the recompute reads the predecessor once more
            self._markers[k] = m
            self.store.put(m.slot, ActivationStore.MARKER, None, 0)
            if self._rec is not None:
                self._rec.markers += 1
            return m
        h = _Handle(t, None, None)
        self._handles[k] = h
        a = self._live(self._act_layer, k)
        if a is not None:
            self._promote(h, a[0])
        return h

    def _promote(self, h, lid):
        """Make h the stored activation of layer lid (raw, or queued for the
        codec at the layer's planned error bound)."""
        eb = self.plan.eb.get(lid) if self.plan is not None else None
        h.layer, h.eb = lid, eb
        t = h.raw
        nbytes = t.numel() * 4
        if self._batch:
            self._per_sample[lid] = nbytes / self._batch
        if self._rec is not None:
            self._rec.raw_bytes += nbytes
        if eb is None:
            self.store.put(lid, ActivationStore.RAW, None, nbytes)
            if self._rec is not None:
                self._rec.stored_bytes += nbytes
            return
        # launch now (side stream, no host sync); the oldest in-flight
        # compressions are finished -- container built, original released --
        # once more than `batch_flush` are in flight, so at most that many
        # raw activations outlive their compression
        params = CodecParams(eb=eb, radius=self.radius, preserve_zeros=self.preserve_zeros)
        # slots 1.. (never the thread's main context, which the decoders use
        # in backward while the last compressions may still be in flight)
        h.job = compress_begin([t], [params], slot_base=1 + self._slot, bit_hints=[self._bits.get(lid)],
                               own_scratch=True)
        self._slot = (self._slot + 1) % (self.batch_flush + 1)
        self._pending.append(h)
        while len(self._pending) > self.batch_flush:
            self._finish(self._pending.pop(0))

    def _finish(self, h):
        (c, rep), = compress_end(h.job, compact=True)
        h.job = None
        h.comp, h.report, h.raw = c, rep, None  # the original activation is released here
        self._bits[h.layer] = c.payload_bits  # next iteration's payload cap hint
        self.store.put(h.layer, ActivationStore.COMPRESSED, c, rep.compressed_bytes)
        self._interval_ratios.setdefault(h.layer, []).append(rep.ratio)
        if self._rec is not None:
            self._rec.stored_bytes += rep.compressed_bytes
            self._rec.compressed[h.layer] = (rep.ratio, h.eb)

    def flush(self):
        """Finish every in-flight compression."""
        pend, self._pending = self._pending, []
        for h in pend:
            self._finish(h)

    def _unpack(self, h):
        import torch

        if isinstance(h, tuple):
            return h[1]
        if isinstance(h, _Marker):
            if h.out is None:
                if h.src is None:
                    raise LifecycleError(f"marker {h.slot!r} already released")
                x = self._unpack(h.src)
                with torch.no_grad():
                    h.out = h.mod(x)
                self.store.pop(h.slot)
                h.src = None
            h.unpacks += 1
            out = h.out
            if h.unpacks >= h.packs:
                h.out = None
            return out
        if h.layer is None:
            return h.raw  # a saved tensor that is not a stored activation
        if h.out is None:
            if h.comp is None and h.raw is None:
                raise LifecycleError(f"activation of {h.layer!r} already released")
            if h.job is not None:
                self._pending.remove(h)
                self._finish(h)
            if h.comp is not None:
                out, nz = decompress_device(h.comp, dtype=torch.float32, check=self._collecting)
                h.out = out.view(h.shape)
                if self._collecting:
                    self._R[h.layer] = nz / out.numel()
                self.store.pop(h.layer)
                h.comp = None
            else:
                h.out = h.raw
                if self._collecting:
                    from .tensor import count_nonzero

                    self._R[h.layer] = count_nonzero(h.raw) / h.raw.numel()
                self.store.pop(h.layer)
                h.raw = None
        h.unpacks += 1
        out = h.out
        if h.unpacks >= h.packs:
            h.out = None
        return out

    # ---- iteration protocol --------------------------------------------------
    @contextlib.contextmanager
    def iteration(self):
        """Wrap forward + backward of one training iteration."""
        import torch

        self._collecting = (self.it + 1) == self.next_collection
        self._act_layer.clear()
        self._handles.clear()
        self._cheap.clear()
        self._markers.clear()
        self._R.clear()
        self._lbar.clear()
        self.store.clear()
        self.store.peak_bytes = 0
        self._rec = IterationRecord(self.it)
        # the consumers' output-gradient hooks (L_bar) exist only in collection
        # iterations: full backward hooks wrap every call of their module
        relus = []
        if self._collecting:
            import torch.nn as nn

            # full backward hooks forbid in-place ops on their modules' outputs:
            # in-place ReLUs run out of place in collection iterations only
            scope = self._model.modules() if self._model is not None else (
                m for mod in self._modules() for m in mod.modules())
            for m in scope:
                if isinstance(m, nn.ReLU) and m.inplace:
                    m.inplace = False
                    relus.append(m)
            for lid, (prod, cons) in self.layers.items():
                self._bwd_hooks.append(cons.register_full_backward_hook(self._bwd_hook(lid)))
        try:
            with torch.autograd.graph.saved_tensors_hooks(self._pack, self._unpack):
                yield self
                self.flush()
        finally:
            for h in self._bwd_hooks:
                h.remove()
            self._bwd_hooks.clear()
            for m in relus:
                m.inplace = True
        self._handles.clear()
        self._act_layer.clear()
        self._cheap.clear()
        self._markers.clear()

    def after_step(self):
        """Call after optimizer.step(): interval boundary -> new plan."""
        self.records.append(self._rec)
        budget = self.config.memory_budget_bytes
        if self._collecting:
            self.plan = self.controller.new_interval(self._collect_stats())
            self.next_collection = (self.it + 1) + self.plan.W
            if budget is not None and self.controller.intervals_planned >= 2:
                self.batch_size = self.plan_batch_size()
            self._interval_ratios = {lid: [] for lid in self.layers}
        if budget is not None and (self.store.peak_bytes + self.fixed_bytes
                                   > budget * (1.0 - self.config.reserve_fraction)):
            self.controller.note_reserve_breach()  # training.py:420-426
        self.it += 1
        self._collecting = False
        return self.plan

    def plan_batch_size(self) -> int:
        """Largest power-of-two batch whose projected activation bytes (per-
        sample cost / observed ratio per layer, plus the input) and the
        model's fixed bytes fit the memory budget minus the reserve
        (controller.choose_batch_size; reference training.py:401-416)."""
        costs = {}
        if self.input_sample_bytes:
            costs["input"] = float(self.input_sample_bytes)
        ratios = {}
        for lid in self.layers:
            if lid in self._per_sample:
                costs[lid] = self._per_sample[lid]
            r = self._interval_ratios.get(lid)
            if r:
                ratios[lid] = sum(r) / len(r)
        return choose_batch_size(costs, ratios, self.config, fixed_bytes=self.fixed_bytes)

    @property
    def reserve_breaches(self) -> int:
        return self.controller.reserve_breach_count

    def _collect_stats(self):
        from .tensor import mean_abs

        ids = list(self.layers)
        N = self._batch or 1
        R = [self._R.get(l, 0.0) for l in ids]
        Lb = [self._lbar.get(l, 0.0) for l in ids]
        M = []
        for l in ids:
            cons = self.layers[l][1]
            st = self.optimizer.state.get(cons.weight, {})
            v = st.get("momentum_buffer")
            M.append(mean_abs(v) if v is not None else 0.0)
        if self.sync_stats:
            R, Lb, M = sync_layer_stats(R, Lb, M, self.dist_group)
        return [LayerTrainingStats(layer_id=l, R=min(1.0, max(0.0, r)), L_bar=lb, M_avg=m, N=N)
                for l, r, lb, m in zip(ids, R, Lb, M)]


def device_memory_budget(device=None, headroom_bytes: int = 0) -> int:
    """Bytes this process may plan against on `device`: what the allocator
    already holds plus what the driver reports free (torch.cuda.mem_get_info),
    minus a headroom -- a value for ControllerConfig.memory_budget_bytes."""
    torch = _lib.torch_cuda()
    free, _total = torch.cuda.mem_get_info(device)
    return int(free + torch.cuda.memory_reserved(device) - headroom_bytes)


def sync_layer_stats(R, L_bar, M_avg, group=None):
    """Average per-layer statistics across data-parallel ranks (identical eb
    everywhere).  No-op without an initialised process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return R, L_bar, M_avg
    world = dist.get_world_size(group)
    if world == 1:
        return R, L_bar, M_avg
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    v = torch.tensor(list(R) + list(L_bar) + list(M_avg), dtype=torch.float64, device=dev)
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    v = (v / world).cpu().tolist()
    k = len(R)
    return v[:k], v[k:2 * k], v[2 * k:]
