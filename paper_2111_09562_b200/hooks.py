"""Per-layer activation compression hooks for PyTorch training.

Mirrors the reference's hook API and storage policy
(/root/reference/pkg/src/actcomp/training.py):

* `ActivationStore` -- per-layer slots RAW / COMPRESSED / MARKER with byte
  accounting, put-once / pop-once (LifecycleError), training.py:105-138.
* `ActivationCompressor` -- the train() hook sites (training.py:259-299
  compress after forward, :335-353 lazy decompress in backward, :351-361
  statistics, :381-418 interval boundary) re-expressed for autograd:
  `torch.autograd.graph.saved_tensors_hooks` pack/unpack.

What is stored.  The reference stores every conv layer's output and
recomputes the cheap layers after it (ReLU, max-pool) from it
(training.py:264-299, 344-347).  One slot per conv CALL, found by following
the conv's output through parameter-free / normalisation modules and
in-place ops up to the first ReLU (dataflow, not module order --
torchvision's Bottleneck calls one ReLU module three times, each call
belongs to a different conv):
* conv -> ReLU (or conv -> BN -> residual add -> ReLU): autograd saves the
  ReLU's output (ReLU backward and the next layer's backward both read it):
  that is the stored activation;
* conv -> training-mode BatchNorm -> ReLU with nothing in between: the
  stored activation is the conv output (BN's saved input, which would
  otherwise stay raw), and the ReLU output is a cheap layer recomputed in
  backward from the decompressed conv output with the forward pass's batch
  statistics -- the reference's policy;
* pooling outputs computed from a stored (or recomputed) activation are
  MARKER slots: recomputed in backward.

Consumer.  The reference's consumer of a conv's stored output is the next
parameterised layer downstream (`_consumer_map`, training.py:154-166); its
momentum (M_avg) and output gradient (L_bar) set the layer's error bound.
Here it is the first Conv2d / Linear whose input is the stored activation
(or a pooling / dropout output derived from it), followed across residual
adds by dataflow; when the dataflow passes through a functional view
(torch.flatten), the next Conv2d / Linear in registration order.

Policy, as in the reference:
* no compression during the first interval (W iterations) -- there is no
  plan yet (training.py:265-266);
* every W iterations the collection iteration measures R (nonzero ratio of
  the stored, i.e. decompressed, activation), L_bar (per-sample max of the
  loss gradient at the consumer's output, un-averaged) and M_avg (mean |v|
  of the consumer's momentum) and asks the controller for the next plan;
* layers whose eb is None (skip set) stay raw.

Packing is asynchronous: a stored activation's compression is launched on a
side stream as soon as it exists (`compress_begin`, no host sync); a
compression is finished (`compress_end`: plan read, exact-size container,
original released) as soon as its chain is done, or -- waiting -- once more
than `batch_flush` are in flight or the raw activations waiting behind the
newest one exceed `inflight_bytes` (default: a quarter of the previous
iteration's raw stored bytes).  The training stream is never ordered
after a compression: the container's decompression in backward waits for
its completion event instead.  Decode faults of the (unsynchronised) backward decompressions
are collected at the end of every iteration and raised as FormatError at
the next iteration's start (one event wait).
Under data parallelism the statistics are averaged across ranks before
planning and N is the global batch, so every rank compresses with the error
bound a single-process run at the same global batch would use.
"""
from __future__ import annotations

import contextlib
import weakref
from dataclasses import dataclass, field

from . import _lib
from .codec import DEFAULT_RADIUS, CodecParams, compress_begin, compress_end, decompress_device
from .controller import AdaptiveController, ControllerConfig, LayerTrainingStats, choose_batch_size
from .errors import FormatError, LifecycleError, ParameterError


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

    def __len__(self):
        return len(self._slots)


def _key(t):
    """identity of one version of a tensor (saved-tensor matching)"""
    return (t.data_ptr(), t._version, tuple(t.shape), tuple(t.stride()))


def _tkey(t):
    """identity of a tensor across in-place updates (dataflow tags)"""
    return (t.data_ptr(), tuple(t.shape), tuple(t.stride()))


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


def _numel(shape) -> int:
    n = 1
    for d in shape:
        n *= d
    return n


class _Handle:
    """One saved fp32 tensor.  Autograd saves a module's output while the op
    runs, before the module's forward hook names it, so every saved tensor
    gets a handle; the dataflow hooks then promote the handle of a stored
    activation to its slot: raw until the pending queue is flushed,
    compressed after.  Handles nobody promotes pass the tensor through."""

    __slots__ = ("layer", "eb", "raw", "comp", "report", "packs", "unpacks", "out", "shape", "ref", "job", "rec",
                 "pos", "pf")

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
        self.rec = None  # (recompute fn, source handle, marker slot): a cheap layer's output, recomputed
        self.pos = -1  # index among this iteration's compressed stored activations (promotion order)
        self.pf = None  # (tensor, event): reconstruction prefetched on the decode stream
        # the tensor's identity: a key (pointer, version, shape, stride) is
        # only unique while the tensor lives -- freed memory is reused
        self.ref = weakref.ref(t)


class _BnRelu:
    """relu(batch_norm(x)) with the forward pass's batch statistics: the
    saved output of the ReLU after a training-mode BatchNorm, recomputed in
    backward from the decompressed conv output (reference recompute_cheap,
    training.py:344-347)."""

    __slots__ = ("scale", "shift")

    def __init__(self, bn, mean, invstd):
        import torch

        with torch.no_grad():
            scale = invstd.float()
            if bn.weight is not None:
                scale = scale * bn.weight.detach().float()
            shift = -mean.float() * scale
            if bn.bias is not None:
                shift = shift + bn.bias.detach().float()
        self.scale, self.shift = scale, shift

    def __call__(self, x):
        import torch

        shape = (1, -1) + (1,) * (x.dim() - 2)
        return torch.relu(torch.addcmul(self.shift.view(shape), x, self.scale.view(shape)))


def _bn_batch_stats(bn, x, out):
    """(mean, invstd) the training-mode BatchNorm `bn` normalised x with: the
    ones its autograd node saved (cuDNN / native kernels), else recomputed."""
    import torch

    g = getattr(out, "grad_fn", None)
    try:
        mean, invstd = g._saved_result1, g._saved_result2
        if mean is not None and invstd is not None and mean.numel() == x.shape[1] == invstd.numel():
            return mean.detach(), invstd.detach()
    except (AttributeError, RuntimeError):
        pass
    with torch.no_grad():
        dims = [0] + list(range(2, x.dim()))
        var, mean = torch.var_mean(x.detach().float(), dim=dims, unbiased=False)
        return mean, torch.rsqrt(var + bn.eps)


@dataclass
class IterationRecord:
    iteration: int
    compressed: dict = field(default_factory=dict)  # slot -> (ratio, eb)
    stored_bytes: int = 0   # CMTZ bytes of compressed slots + raw bytes of the others
    device_bytes: int = 0   # device memory the stored containers really hold (incl. the decode index)
    raw_bytes: int = 0
    markers: int = 0        # cheap-layer outputs recomputed instead of stored
    slots: list = field(default_factory=list)  # stored-activation slots in forward order


class _LayerMap(dict):
    """conv_layer_map's result: {layer_id: (producer module, consumer module
    or None)} plus the model it came from."""

    def __init__(self, d, model):
        super().__init__(d)
        self.model = model


def _is_relu(m):
    import torch.nn as nn

    return isinstance(m, (nn.ReLU, nn.ReLU6, nn.LeakyReLU))


def _is_param_layer(m):
    import torch.nn as nn

    return isinstance(m, (nn.Conv1d, nn.Conv2d, nn.Conv3d, nn.Linear))


def _passes_tags(m):
    """modules a producer tag flows through on its way to the ReLU (and a
    consumer tag on its way to the next parameterised layer): parameter-free
    leaves and normalisations"""
    import torch.nn as nn

    if isinstance(m, nn.modules.batchnorm._NormBase):
        return True
    return not any(True for _ in m.parameters(recurse=False))


class ActivationCompressor:
    """Adaptive activation compression for a PyTorch model.

    layers: `conv_layer_map(model)` (every Conv2d of the model is a producer;
    stored activations and consumers are found by dataflow), or an explicit
    {layer_id: (producer_module, consumer_module or None)} map -- a producer
    that is itself a ReLU stores its own output.
    """

    def __init__(self, layers, optimizer, config: ControllerConfig | None = None, radius: int = DEFAULT_RADIUS,
                 preserve_zeros: bool = True, grad_scale=None, batch_flush: int = 8, dist_group=None,
                 sync_stats: bool = True, input_sample_bytes: float | None = None, fixed_bytes: float | None = None,
                 recompute_cheap: bool = True, codec_on_compute_stream: bool = False,
                 prefetch_decode: bool = False, inflight_bytes: int | None = None):
        import torch.nn as nn

        self.layers = dict(layers)
        self._model = getattr(layers, "model", None)
        self.optimizer = optimizer
        self.config = config or ControllerConfig()
        self.controller = AdaptiveController(self.config)
        self.radius = radius
        self.preserve_zeros = preserve_zeros
        self.grad_scale = grad_scale  # None: use the batch size (mean-reduced loss)
        # at most `batch_flush` compressions in flight (each holds a side
        # stream + library context), and the raw activations of all but the
        # newest below `inflight_bytes`: the host runs ahead of the GPU by
        # that much instead of waiting for each compression
        # inflight_bytes None: a quarter of the previous iteration's raw stored
        # bytes (0 -- one compression at a time -- until an iteration is seen),
        # so a model with few large activations keeps its forward peak while
        # one with many (ResNet-50: 49 per iteration) overlaps compressions
        self.batch_flush = batch_flush
        self.inflight_bytes = inflight_bytes
        self._pending_bytes = 0
        self.dist_group = dist_group
        self.sync_stats = sync_stats
        self.recompute_cheap = recompute_cheap
        # compressions in order on the training stream (no SM contention with
        # the convolutions) instead of side streams
        self.codec_on_compute_stream = codec_on_compute_stream
        # backward: while one stored activation is reconstructed for autograd,
        # the one stored before it (the next one backward needs) is decoded
        # on a side stream, overlapping the decoder with backward's kernels
        self.prefetch_decode = prefetch_decode
        self._pf_stream = None
        self._order: list = []  # this iteration's compressed stored activations, promotion order
        self.plan = None
        self.it = 0
        self.next_collection = self.controller.W
        self.store = ActivationStore()
        self.records: list[IterationRecord] = []
        # per-iteration dataflow state
        self._act_layer: dict = {}   # key -> (slot, ref): stored activations by tensor version
        self._handles: dict = {}     # key -> _Handle
        self._ptag: dict = {}        # tkey -> (slot, ref): a producer's output on its way to the ReLU
        self._ctag: dict = {}        # tkey -> (slot, ref): a stored activation on its way to its consumer
        self._cheap: dict = {}
        self._markers: dict = {}
        self._bnp: dict = {}         # tkey -> (slot, bn, conv-output ref, output version, fn, ref): a BN output on its way to the ReLU
        self._slot_out: dict = {}    # slot -> weakref of its producer's output
        self._calls: dict = {}       # layer id -> calls this iteration
        self._await_consumer: list = []  # slots stored this iteration without a consumer yet
        self._pending: list[_Handle] = []  # compressions launched, not yet synchronised (oldest first)
        self._slot = 0
        self._collecting = False
        self._R: dict[str, float] = {}
        self._lbar: dict[str, float] = {}
        self._bits: dict[str, tuple] = {}
        self._batch = None
        self._rec = None
        self._status = None          # decode-fault collection of the previous iteration
        self._capture = None         # slots whose (input, container) the next iteration keeps
        self.captured: dict = {}     # slot -> (host fp32 copy of the stored activation, container)
        # slot -> consumer module; explicit consumers from the map, the rest by dataflow
        self.consumers: dict = {}
        self._slot_layer: dict = {}  # slot -> layer id
        self._hooks = []
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
        self._interval_ratios: dict[str, list] = {}

        self._producer: dict = {}   # id(module) -> layer id
        self._explicit_consumer: dict = {}
        for lid, (prod, cons) in self.layers.items():
            self._producer[id(prod)] = lid
            if cons is not None:
                self._explicit_consumer[lid] = cons
        # registration-order fallback consumer (reference _consumer_map):
        # the next Conv/Linear after the producer
        leaves = self._leaf_modules()
        self._fallback_consumer: dict = {}
        for i, (_, m) in enumerate(leaves):
            lid = self._producer.get(id(m))
            if lid is None:
                continue
            for _, m2 in leaves[i + 1:]:
                if _is_param_layer(m2):
                    self._fallback_consumer[lid] = m2
                    break
        seen = set()
        for _, m in leaves:
            if id(m) in seen:
                continue
            seen.add(id(m))
            self._hooks.append(m.register_forward_hook(self._leaf_hook))
        self._pools = (nn.MaxPool1d, nn.MaxPool2d, nn.MaxPool3d, nn.AvgPool1d, nn.AvgPool2d, nn.AvgPool3d)

    # ---- construction helpers -------------------------------------------
    @staticmethod
    def conv_layer_map(model):
        """{name: (conv module, None)} for every Conv2d of the model: the
        stored activation and the consumer of each call are found by
        dataflow (training.py:154-166, 264-283)."""
        import torch.nn as nn

        return _LayerMap({n: (m, None) for n, m in model.named_modules() if isinstance(m, nn.Conv2d)}, model)

    def _leaf_modules(self):
        if self._model is not None:
            return [(n, m) for n, m in self._model.named_modules() if not list(m.children())]
        out = []
        for lid, (prod, cons) in self.layers.items():
            out.append((lid, prod))
            if cons is not None:
                out.append((lid + ".consumer", cons))
        return out

    def remove(self):
        for h in self._hooks:
            h.remove()
        self._hooks.clear()

    # ---- dataflow --------------------------------------------------------
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

    def _new_slot(self, lid):
        k = self._calls.get(lid, 0)
        self._calls[lid] = k + 1
        slot = lid if k == 0 else f"{lid}#{k}"
        self._slot_layer[slot] = lid
        return slot

    def _leaf_hook(self, mod, inp, out):
        import torch
        import torch.nn as nn

        if not torch.is_tensor(out):
            return
        x = inp[0] if inp and torch.is_tensor(inp[0]) else None
        if x is not None and _is_param_layer(mod):
            self._match_consumer(mod, x, out)
        lid = self._producer.get(id(mod))
        if lid is not None:
            if self._batch is None and x is not None and x.dim() > 0:
                self._batch = int(x.shape[0])
            slot = self._new_slot(lid)
            if _is_relu(mod):
                self._store(slot, out)
            else:
                self._ptag[_tkey(out)] = (slot, weakref.ref(out))
                self._slot_out[slot] = weakref.ref(out)
            return
        if x is None:
            return
        k = _tkey(x)
        pt = self._live(self._ptag, k)
        if pt is not None:
            if _is_relu(mod):
                del self._ptag[k]
                if not self._store_bn_relu(pt[0], mod, x, out):
                    self._store(pt[0], out)
                return
            if _passes_tags(mod):
                self._ptag[_tkey(out)] = (pt[0], weakref.ref(out))
                if (self.recompute_cheap and isinstance(mod, nn.modules.batchnorm._BatchNorm) and mod.training
                        and self._is_producer_output(pt[0], x)):
                    self._bnp[_tkey(out)] = (pt[0], mod, weakref.ref(x), out._version,
                                             _BnRelu(mod, *_bn_batch_stats(mod, x, out)), weakref.ref(out))
        ct = self._live(self._ctag, k)
        if ct is not None and not _is_param_layer(mod) and _passes_tags(mod):
            self._ctag[_tkey(out)] = (ct[0], weakref.ref(out))
        if self.recompute_cheap and isinstance(mod, self._pools):
            src = self._live(self._handles, _key(x))
            if src is not None and (src.layer is not None or src.rec is not None):
                self._cheap[_key(out)] = (type(mod).__name__.lower(), mod, src, weakref.ref(out))

    def _is_producer_output(self, slot, x):
        """x is the producer's own output (conv -> BN directly, nothing between)"""
        return self._slot_out.get(slot) is not None and self._slot_out[slot]() is x

    def _store_bn_relu(self, slot, relu, x, out):
        """conv -> training-mode BatchNorm -> ReLU, the BN output untouched in
        between (no residual add): the stored activation is the conv output
        (BN's saved input -- stored instead of raw) and the ReLU output is a
        cheap layer, recomputed in backward from the decompressed conv output
        with the forward pass's batch statistics (reference MARKER slots,
        training.py:295-296, 344-347).  False: not that pattern."""
        bnp = self._live(self._bnp, _tkey(x))
        if bnp is None or bnp[0] != slot:
            return False
        inplace = out is x
        if x._version != bnp[3] + (1 if inplace else 0):
            return False  # modified between the BN and the ReLU (e.g. a residual add)
        conv_out = bnp[2]()
        if conv_out is None:
            return False
        self._store(slot, conv_out)
        src = self._live(self._handles, _key(conv_out))
        if src is None or src.layer != slot:
            return True  # not saved by the BN (eval-like use): only the conv output is stored
        fn = bnp[4]
        mslot = f"relu@{slot}"
        self._ctag[_tkey(out)] = (slot, weakref.ref(out))  # the consumer search continues past the ReLU
        h = self._live(self._handles, _key(out))
        if h is not None and h.layer is None and h.rec is None:
            # the ReLU saved its output while it ran: that handle recomputes
            h.rec = (fn, src, mslot)
            h.raw = None
            src.packs += 1
            self.store.put(mslot, ActivationStore.MARKER, None, 0)
            if self._rec is not None:
                self._rec.markers += 1
        else:
            # saved later (by the consumer): the pack makes the marker
            self._cheap[_key(out)] = ("relu", fn, src, weakref.ref(out))
        return True

    def _store(self, slot, out):
        """`out` is the stored activation of `slot` (saved by its op before
        this hook ran, or saved later by its consumer)."""
        k = _key(out)
        self._act_layer[k] = (slot, weakref.ref(out))
        self._ctag[_tkey(out)] = (slot, weakref.ref(out))
        if self._rec is not None:
            self._rec.slots.append(slot)
        lid = self._slot_layer[slot]
        cons = self._explicit_consumer.get(lid)
        if cons is not None:
            self.consumers[slot] = cons
        elif slot not in self.consumers or self._collecting:
            self._await_consumer.append(slot)
        h = self._live(self._handles, k)
        if h is not None and h.layer is None:
            self._promote(h, slot)

    def _match_consumer(self, mod, x, out):
        """mod (a Conv/Linear) consumes x: the consumer of every waiting slot
        whose activation reaches it by dataflow, or whose registration-order
        fallback it is."""
        if not self._await_consumer:
            return
        ct = self._live(self._ctag, _tkey(x))
        hit = []
        for slot in self._await_consumer:
            if (ct is not None and ct[0] == slot) or self._fallback_consumer.get(self._slot_layer[slot]) is mod:
                hit.append(slot)
        for slot in hit:
            self._await_consumer.remove(slot)
            self.consumers[slot] = mod
            if self._collecting:
                self._watch_grad(slot, out)

    def _watch_grad(self, slot, out):
        """L_bar of `slot`: per-sample max |g| of the loss gradient at its
        consumer's output (training.py:358-361), un-averaged."""
        if not getattr(out, "requires_grad", False):
            return

        def hook(g):
            from .tensor import per_sample_max

            scale = self.grad_scale if self.grad_scale is not None else (self._batch or 1)
            _, lbar = per_sample_max(g.detach().float())
            self._lbar[slot] = lbar * scale

        out.register_hook(hook)

    # ---- saved-tensor hooks ------------------------------------------------
    def _pack(self, t):
        import torch

        if t.dtype != torch.float32 or isinstance(t, torch.nn.Parameter):
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
        if cheap is not None and (cheap[2].layer is not None or cheap[2].rec is not None):
            # (the source handle -- a stored or recomputed activation of this
            # iteration -- is valid whether or not its tensor object is
            # still alive: a finished compression has released it)
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

    def _promote(self, h, slot):
        """Make h the stored activation of `slot` (raw, or queued for the
        codec at the slot's planned error bound)."""
        eb = self.plan.eb.get(slot) if self.plan is not None else None
        h.layer, h.eb = slot, eb
        t = h.raw
        nbytes = t.numel() * 4
        if self._batch:
            self._per_sample[slot] = nbytes / self._batch
        if self._rec is not None:
            self._rec.raw_bytes += nbytes
        if eb is None:
            self.store.put(slot, ActivationStore.RAW, None, nbytes)
            if self._rec is not None:
                self._rec.stored_bytes += nbytes
                self._rec.device_bytes += nbytes
            return
        if not t.is_cuda:
            raise ParameterError(f"activation of {slot!r} is not on a CUDA device: the codec has no CPU path")
        # launch now (side stream, no host sync); the oldest in-flight
        # compressions are finished -- container built, original released --
        # once more than `batch_flush` are in flight, so at most that many
        # raw activations outlive their compression
        params = CodecParams(eb=eb, radius=self.radius, preserve_zeros=self.preserve_zeros)
        hb, ho = self._hint(slot, eb)
        # slots 1.. (never the thread's main context, which the decoders use
        # in backward while the last compressions may still be in flight)
        h.job = compress_begin([t], [params], slot_base=1 + self._slot, bit_hints=[hb], outlier_hints=[ho],
                               own_scratch=True, on_caller_stream=self.codec_on_compute_stream)
        h.pos = len(self._order)
        self._order.append(h)
        self._slot = (self._slot + 1) % (self.batch_flush + 1)
        self._pending.append(h)
        self._pending_bytes += nbytes
        # finish what is already done without waiting; wait only when more
        # than batch_flush are in flight (their contexts are reused next) or
        # the older raw activations exceed inflight_bytes
        limit = self.inflight_bytes
        if limit is None:
            limit = self.records[-1].raw_bytes // 4 if self.records else 0
        while self._pending and (len(self._pending) > self.batch_flush or self._pending[0].job.ready()
                                 or (len(self._pending) > 1 and self._pending_bytes > limit)):
            self._finish(self._pending.pop(0))

    def _hint(self, slot, eb):
        """Cap hints (payload bits, outlier count) for `slot` from its last
        compression.  The payload hint only holds at the same error bound: a
        new plan changes the eb and with it the payload size (a smaller eb
        can need far more than 1.25x the old bits), and an overflowing cap
        means a synchronous re-compression, so a new eb starts from the safe
        n*ceil(log2 L) cap.  The outlier count is scaled by the eb ratio
        when the eb shrank (the tail beyond the radius grows)."""
        prev = self._bits.get(slot)
        if prev is None:
            return None, None
        peb, bits, nout = prev
        if peb == eb:
            return bits, nout
        return None, int(nout * max(1.0, peb / eb)) if nout else None

    def capture_next_iteration(self, slots=None):
        """Keep, for the next iteration, a host copy of every compressed
        stored activation (or of `slots`) and its container, in `captured`
        -- the per-layer spot check of training tensors against the
        reference codec (per-layer ratio/eb vs oracle)."""
        self._capture = set(slots) if slots is not None else True
        self.captured = {}

    def _finish(self, h):
        self._pending_bytes -= 4 * _numel(h.shape)
        # order=False: the training stream never waits for a compression;
        # the container's readers (the backward decompression) do
        (c, rep), = compress_end(h.job, compact=True, order=False)
        h.job = None
        if self._capture is True or (self._capture and h.layer in self._capture):
            self.captured[h.layer] = (h.raw.detach().cpu().numpy(), c, h.eb)  # shaped: CMTZ records the dims
        h.comp, h.report, h.raw = c, rep, None  # the original activation is released here
        self._bits[h.layer] = (h.eb, c.payload_bits, c._n_outliers)  # next iteration's cap hints
        self.store.put(h.layer, ActivationStore.COMPRESSED, c, rep.compressed_bytes)
        self._interval_ratios.setdefault(h.layer, []).append(rep.ratio)
        if self._rec is not None:
            self._rec.stored_bytes += rep.compressed_bytes
            self._rec.device_bytes += c.device_nbytes
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
        if h.rec is not None:
            # a cheap layer's output: recomputed once from its stored source
            if h.out is None:
                fn, src, mslot = h.rec
                if src is None:
                    raise LifecycleError(f"recomputed output {mslot!r} already released")
                x = self._unpack(src)
                with torch.no_grad():
                    h.out = fn(x)
                self.store.pop(mslot)
                h.rec = (fn, None, mslot)
            h.unpacks += 1
            out = h.out
            if h.unpacks >= h.packs:
                h.out = None
            return out
        if h.layer is None:
            return h.raw  # a saved tensor that is not a stored activation
        if h.out is None and h.pf is not None:
            # decoded ahead on the prefetch stream
            out, ev = h.pf
            h.pf = None
            cur = _lib.current_stream()
            cur.wait_event(ev)
            out.record_stream(cur)
            h.out = out.view(h.shape)
            self.store.pop(h.layer)
            h.comp = None
            self._prefetch_before(h)
        if h.out is None:
            if h.comp is None and h.raw is None:
                raise LifecycleError(f"activation of {h.layer!r} already released")
            if h.job is not None:
                self._pending.remove(h)
                self._finish(h)
            if h.comp is not None:
                # collection iterations read R back at once; otherwise the
                # decode status is collected at the end of the iteration
                out, nz = decompress_device(h.comp, dtype=torch.float32, check=self._collecting,
                                            count_nonzero=self._collecting)
                h.out = out.view(h.shape)
                if self._collecting:
                    self._R[h.layer] = nz / out.numel()
                self.store.pop(h.layer)
                h.comp = None
                self._prefetch_before(h)
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

    def _prefetch_before(self, h):
        """Launch the decode of the compressed activation stored just before
        h (backward's next one) on the prefetch stream, its own library
        context; not in collection iterations (they read R back at once)."""
        import torch

        if not self.prefetch_decode or self._collecting or h.pos <= 0:
            return
        g = self._order[h.pos - 1]
        if g.comp is None or g.out is not None or g.pf is not None or g.unpacks or g.job is not None:
            return
        cur = _lib.current_stream()
        if self._pf_stream is None:
            self._pf_stream = torch.cuda.Stream(device=cur.device)
        ps = self._pf_stream
        ps.wait_stream(cur)  # after the caller's queued work (memory the allocator handed back)
        out, _ = decompress_device(g.comp, dtype=torch.float32, stream=ps, check=False, count_nonzero=False,
                                   slot=self.batch_flush + 2)
        g.pf = (out, ps.record_event())

    # ---- iteration protocol --------------------------------------------------
    def _reset_iteration_state(self):
        for d in (self._act_layer, self._handles, self._ptag, self._ctag, self._cheap, self._markers, self._calls,
                  self._bnp, self._slot_out):
            d.clear()
        for h in self._order:
            if h.pf is not None:  # decoded ahead but never read back: join its stream
                cur = _lib.current_stream()
                cur.wait_event(h.pf[1])
                h.pf[0].record_stream(cur)
                h.pf = None
        self._order = []
        self._await_consumer = []

    @contextlib.contextmanager
    def iteration(self):
        """Wrap forward + backward of one training iteration."""
        import torch

        if self._status is not None:
            # decode faults of the previous iteration's backward (reference
            # decompress raises FormatError, codec.py:356-359)
            tok, self._status = self._status, None
            if _lib.decode_status_result(tok):
                raise FormatError("invalid code in a stored activation's bitstream "
                                  "(or outlier markers disagree with stored indices)")
        self._collecting = (self.it + 1) == self.next_collection
        self._reset_iteration_state()
        # the same slot (side stream + library context) for the same stored
        # activation every iteration: each context's scratch reaches its
        # size once, no allocation (device-wide synchronisation) later
        self._slot = 0
        self._batch = None  # taken from this iteration's first producer input
        self._R.clear()
        self._lbar.clear()
        self.store.clear()
        self.store.peak_bytes = 0
        self._rec = IterationRecord(self.it)
        try:
            with torch.autograd.graph.saved_tensors_hooks(self._pack, self._unpack):
                yield self
                self.flush()
        finally:
            self._reset_iteration_state()
            if self.captured:
                self._capture = None
        if self.plan is not None and _lib.cuda_available():
            self._status = _lib.take_decode_status()

    def after_step(self):
        """Call after optimizer.step(): interval boundary -> new plan."""
        self.records.append(self._rec)
        budget = self.config.memory_budget_bytes
        if self._collecting:
            self.plan = self.controller.new_interval(self._collect_stats())
            self.next_collection = (self.it + 1) + self.plan.W
            if budget is not None and self.controller.intervals_planned >= 2:
                self.batch_size = self.plan_batch_size()
            self._interval_ratios = {}
        if budget is not None and (self.store.peak_bytes + self.fixed_bytes
                                   > budget * (1.0 - self.config.reserve_fraction)):
            self.controller.note_reserve_breach()  # training.py:420-426
        self.it += 1
        self._collecting = False
        return self.plan

    def plan_batch_size(self) -> int:
        """Largest power-of-two batch whose projected activation bytes (per-
        sample cost / observed ratio per slot, plus the input) and the
        model's fixed bytes fit the memory budget minus the reserve
        (controller.choose_batch_size; reference training.py:401-416)."""
        costs = {}
        if self.input_sample_bytes:
            costs["input"] = float(self.input_sample_bytes)
        ratios = {}
        for slot, cost in self._per_sample.items():
            costs[slot] = cost
            r = self._interval_ratios.get(slot)
            if r:
                ratios[slot] = sum(r) / len(r)
        return choose_batch_size(costs, ratios, self.config, fixed_bytes=self.fixed_bytes)

    @property
    def reserve_breaches(self) -> int:
        return self.controller.reserve_breach_count

    def _collect_stats(self):
        from .tensor import mean_abs

        ids = list(self._rec.slots) if self._rec is not None else []
        world = 1
        if self.sync_stats:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized():
                world = dist.get_world_size(self.dist_group)
        # DDP averages the ranks' gradients: the error model's N is the
        # global batch (a single-process run at that batch plans the same eb)
        N = (self._batch or 1) * world
        R = [self._R.get(s, 0.0) for s in ids]
        Lb = [self._lbar.get(s, 0.0) for s in ids]
        M = []
        for s in ids:
            cons = self.consumers.get(s)
            v = None
            w = getattr(cons, "weight", None) if cons is not None else None
            if w is not None:
                v = self.optimizer.state.get(w, {}).get("momentum_buffer")
            M.append(mean_abs(v) if v is not None else 0.0)
        if self.sync_stats:
            R, Lb, M = sync_layer_stats(R, Lb, M, self.dist_group)
        return [LayerTrainingStats(layer_id=s, R=min(1.0, max(0.0, r)), L_bar=lb, M_avg=m, N=N)
                for s, r, lb, m in zip(ids, R, Lb, M)]

    def consumer_names(self) -> dict:
        """slot -> qualified name of its consumer module (after a forward)."""
        names = {id(m): n for n, m in (self._model.named_modules() if self._model is not None else [])}
        return {s: names.get(id(m), type(m).__name__) for s, m in self.consumers.items()}


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
