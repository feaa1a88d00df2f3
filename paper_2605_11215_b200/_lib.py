"""ctypes binding of librcv.so (include/rcv.h) plus thin tensor-level helpers.

This is the only place the package touches the native library.  There is no
CPU fallback: if the library is missing, or a data-plane call is made on a
tensor that is not on a CUDA device, the call raises.
"""

from __future__ import annotations

import ctypes
import os
from collections import OrderedDict
from typing import Optional, Sequence

import torch

F32, F64, BF16 = 0, 1, 2
OP_CANON = 0x40
VARIANT_AUTO, VARIANT_TMA, VARIANT_DIRECT, VARIANT_SCALAR = 0, 1, 2, 3
MAX_IN = 64
MAX_OUT = 64

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librcv.so")

# every symbol include/rcv.h declares (tests check the export table)
EXPORTS = (
    "rcv_last_error", "rcv_version", "rcv_launch_count", "rcv_device_count",
    "rcv_enable_peer_access", "rcv_fold", "rcv_masked_allreduce",
    "rcv_masked_allreduce_multidev", "rcv_accumulate", "rcv_tree_commit",
    "rcv_tree_program", "rcv_copy", "rcv_zero", "rcv_compare",
    "rcv_sgd_commit", "rcv_unit_lanes", "rcv_toy_grad",
    "rcv_ipc_export", "rcv_ipc_import", "rcv_barrier", "rcv_tree_commit_at",
    "rcv_ctx_create", "rcv_ctx_destroy", "rcv_ctx_finish", "rcv_ctx_set_timing",
    "rcv_ctx_timing", "rcv_plan_create", "rcv_plan_destroy", "rcv_plan_bucket",
    "rcv_vmm_alloc", "rcv_vmm_import", "rcv_kacc_push", "rcv_ctx_set_liveness", "rcv_ctx_poll",
    "rcv_liveness_create", "rcv_liveness_dead_word", "rcv_liveness_decide",
    "rcv_liveness_stats", "rcv_liveness_note_kill", "rcv_liveness_destroy",
    "rcv_mc_supported", "rcv_mc_granularity", "rcv_mc_create", "rcv_mc_import",
    "rcv_mc_add_device", "rcv_mc_bind", "rcv_mc_map", "rcv_mc_release",
    "rcv_pool_sets",
)


class RcvError(RuntimeError):
    """A librcv.so call returned an error code."""


class _Block(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("lo", ctypes.c_uint32),
                ("level", ctypes.c_uint32), ("dtype", ctypes.c_int)]


class PlanDesc(ctypes.Structure):
    """rcv_plan_desc (include/rcv.h)."""
    _fields_ = [
        ("n_pre", ctypes.c_int), ("pre_blocks", ctypes.POINTER(_Block)),
        ("pre_counts", ctypes.POINTER(ctypes.c_int)),
        ("pre_leaves", ctypes.POINTER(ctypes.c_uint32)),
        ("pre_out", ctypes.POINTER(ctypes.c_void_p)), ("set_stride", ctypes.c_size_t),
        ("n_comb", ctypes.c_int), ("comb_blocks", ctypes.POINTER(_Block)),
        ("comb_rank", ctypes.POINTER(ctypes.c_int)),
        ("n_leaves", ctypes.c_uint32), ("n_comb_out", ctypes.c_int),
        ("comb_out", ctypes.POINTER(ctypes.c_void_p)),
        ("slice_q", ctypes.c_int), ("slice_nr", ctypes.c_int),
        ("n_bcast", ctypes.c_int), ("bcast_src", ctypes.c_void_p),
        ("bcast_out", ctypes.POINTER(ctypes.c_void_p)),
        ("acc_dtype", ctypes.c_int), ("divisor", ctypes.c_double),
        ("variant", ctypes.c_int), ("comb_variant", ctypes.c_int),
        ("live_mask", ctypes.c_uint64), ("participate", ctypes.c_int),
        ("remote_in", ctypes.c_int), ("remote_out", ctypes.c_int),
        ("guarded", ctypes.c_int), ("comb_out_mc", ctypes.c_uint32),
    ]


_lib: Optional[ctypes.CDLL] = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RcvError(
            "librcv.so not built (%s); run __graft_entry__.build() or "
            "`make -C paper_2605_11215_b200/csrc`" % LIB_PATH)
    lib = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, u64, u32 = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                             ctypes.c_uint64, ctypes.c_uint32)
    pvp = ctypes.POINTER(ctypes.c_void_p)
    sig = {
        "rcv_last_error": (ctypes.c_char_p, []),
        "rcv_version": (i32, []),
        "rcv_launch_count": (ctypes.c_ulonglong, []),
        "rcv_device_count": (i32, [ctypes.POINTER(i32)]),
        "rcv_enable_peer_access": (i32, [i32, ctypes.POINTER(i32)]),
        "rcv_fold": (i32, [i32, pvp, ctypes.POINTER(ctypes.c_uint8),
                           ctypes.POINTER(i32), i32, pvp, i32, sz,
                           ctypes.c_double, i32, vp]),
        "rcv_masked_allreduce": (i32, [pvp, i32, u64, i32, sz,
                                       ctypes.c_double, vp]),
        "rcv_masked_allreduce_multidev": (i32, [pvp, i32, u64, i32, sz,
                                                ctypes.c_double, i32,
                                                ctypes.POINTER(i32), pvp]),
        "rcv_accumulate": (i32, [vp, vp, i32, i32, sz, i32, vp]),
        "rcv_tree_commit": (i32, [ctypes.POINTER(_Block), i32, u32, i32, pvp,
                                  i32, sz, ctypes.c_double, i32, vp]),
        "rcv_tree_program": (i32, [ctypes.POINTER(u32), ctypes.POINTER(u32),
                                   i32, u32, ctypes.POINTER(ctypes.c_uint8),
                                   ctypes.POINTER(i32)]),
        "rcv_copy": (i32, [vp, vp, sz, vp]),
        "rcv_zero": (i32, [vp, sz, vp]),
        "rcv_compare": (i32, [vp, vp, sz, vp, vp]),
        "rcv_sgd_commit": (i32, [vp, vp, i32, sz, ctypes.c_double,
                                 ctypes.c_double, vp]),
        "rcv_unit_lanes": (i32, [vp, u64, sz, ctypes.c_double,
                                 ctypes.c_double, i32, vp]),
        "rcv_toy_grad": (i32, [i32, vp, vp, vp, sz, vp, vp, vp]),
        "rcv_ipc_export": (i32, [vp, vp, ctypes.POINTER(sz)]),
        "rcv_ipc_import": (i32, [vp, sz, ctypes.POINTER(vp)]),
        "rcv_barrier": (i32, [vp, pvp, i32, i32, u64, u64, u64, vp, vp]),
        "rcv_tree_commit_at": (i32, [ctypes.POINTER(_Block), i32, u32, i32, pvp,
                                     i32, sz, sz, sz, ctypes.c_double, i32, vp]),
        "rcv_ctx_create": (i32, [i32, i32, vp, pvp, vp, u64, ctypes.POINTER(vp)]),
        "rcv_pool_sets": (i32, []),
        "rcv_ctx_destroy": (i32, [vp]),
        "rcv_ctx_finish": (i32, [vp, u64, i32, vp]),
        "rcv_ctx_set_timing": (i32, [vp, i32]),
        "rcv_ctx_timing": (i32, [vp, i32, ctypes.POINTER(i32), ctypes.POINTER(ctypes.c_float),
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i32)]),
        "rcv_plan_create": (i32, [vp, ctypes.POINTER(PlanDesc), ctypes.POINTER(vp)]),
        "rcv_plan_destroy": (i32, [vp]),
        "rcv_plan_bucket": (i32, [vp, sz, sz, vp]),
        "rcv_vmm_alloc": (i32, [sz, ctypes.POINTER(vp), ctypes.POINTER(sz), ctypes.POINTER(i32)]),
        "rcv_vmm_import": (i32, [i32, sz, i32, ctypes.POINTER(vp)]),
        "rcv_kacc_push": (i32, [pvp, ctypes.POINTER(u64), ctypes.POINTER(u64), i32, i32,
                                pvp, i32, vp, sz, vp]),
        "rcv_ctx_set_liveness": (i32, [vp, vp]),
        "rcv_ctx_poll": (i32, [vp, u64, i32, vp]),
        "rcv_liveness_create": (i32, [ctypes.c_char_p, i32, i32, u64, u64, ctypes.POINTER(vp)]),
        "rcv_liveness_dead_word": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(u32)]),
        "rcv_liveness_decide": (i32, [vp, u64, ctypes.POINTER(u32), ctypes.POINTER(u64)]),
        "rcv_liveness_stats": (i32, [vp, i32, ctypes.POINTER(u64), ctypes.POINTER(u64),
                                     ctypes.POINTER(u64), ctypes.POINTER(u64)]),
        "rcv_liveness_note_kill": (i32, [vp]),
        "rcv_liveness_destroy": (i32, [vp, i32]),
        "rcv_mc_supported": (i32, [ctypes.POINTER(i32)]),
        "rcv_mc_granularity": (i32, [i32, ctypes.POINTER(sz)]),
        "rcv_mc_create": (i32, [sz, i32, ctypes.POINTER(u64), ctypes.POINTER(sz),
                                ctypes.POINTER(i32)]),
        "rcv_mc_import": (i32, [i32, ctypes.POINTER(u64)]),
        "rcv_mc_add_device": (i32, [u64]),
        "rcv_mc_bind": (i32, [u64, vp, sz]),
        "rcv_mc_map": (i32, [u64, sz, ctypes.POINTER(vp)]),
        "rcv_mc_release": (i32, [u64, vp, sz]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = load().rcv_last_error().decode(errors="replace")
        raise RcvError("librcv error %d: %s" % (rc, msg))


# ---- tensor helpers --------------------------------------------------------

_DT = {torch.float32: F32, torch.float64: F64, torch.bfloat16: BF16}


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError("unsupported dtype %s (float32/float64/bfloat16)"
                        % t.dtype) from None


def require_cuda(t: torch.Tensor, what: str = "tensor") -> None:
    if not isinstance(t, torch.Tensor):
        raise TypeError("%s must be a torch.Tensor on a CUDA device, got %r"
                        % (what, type(t).__name__))
    if not t.is_cuda:
        raise RcvError("%s is on %s: the data plane runs only on CUDA devices "
                       "(no CPU fallback)" % (what, t.device))
    if t.dim() != 1 or not t.is_contiguous():
        raise ValueError("%s must be a contiguous 1-D view" % what)


def raw_stream(device_index: int) -> int:
    """The current stream of a CUDA device as a cudaStream_t (an int); the
    raw accessor skips building a torch.cuda.Stream per call (host time of
    the small-bucket collective)."""
    return torch._C._cuda_getCurrentRawStream(device_index)


def stream_of(t: torch.Tensor) -> int:
    return raw_stream(t.device.index)


def _ptrs(ts: Sequence[torch.Tensor]):
    arr = (ctypes.c_void_p * max(1, len(ts)))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr()
    return arr


def fold(inputs: Sequence[torch.Tensor], ops: Sequence[int],
         outputs: Sequence[torch.Tensor], divisor: float = 0.0,
         variant: int = VARIANT_AUTO, stream: Optional[int] = None) -> None:
    """rcv_fold over torch tensors (all on one device, same numel)."""
    if not outputs:
        return
    acc = outputs[0]
    for t in list(inputs) + list(outputs):
        require_cuda(t)
        if t.numel() != acc.numel():
            raise ValueError("fold operands differ in length")
    n_in = len(inputs)
    opa = (ctypes.c_uint8 * max(1, n_in))(*ops)
    dta = (ctypes.c_int * max(1, n_in))(*[dtype_code(t) for t in inputs])
    _check(load().rcv_fold(n_in, _ptrs(inputs), opa, dta, len(outputs),
                           _ptrs(outputs), dtype_code(acc), acc.numel(),
                           float(divisor), variant,
                           stream if stream is not None else stream_of(acc)))


# prepared arguments of the drop-in collective by call signature (every
# view's address, length, dtype and stride, the contributor mask): a bucket
# reduced again (every step, every re-reduce) skips validation and argument
# marshalling (host time of the small-bucket collective)
_ar_cache: "OrderedDict" = OrderedDict()


class _ArgsAR:
    __slots__ = ("multi", "ptrs", "n", "code", "numel", "devs", "dev_arr", "first_dev")


def _prepare_allreduce(views, n, mask):
    first = views[0]
    for v in views:
        require_cuda(v, "bucket view")
        if v.dtype != first.dtype or v.numel() != first.numel():
            raise ValueError("bucket views differ in dtype or length")
    code = dtype_code(first)
    if code == BF16:
        raise TypeError("bucket views hold accumulators: float32 or float64")
    a = _ArgsAR()
    a.ptrs, a.n, a.code, a.numel = _ptrs(views), n, code, first.numel()
    a.devs = sorted({v.device.index for v in views})
    a.multi = len(a.devs) > 1
    a.first_dev = first.device.index
    if a.multi:
        enable_peer_access(a.devs)
        a.dev_arr = (ctypes.c_int * len(a.devs))(*a.devs)
    return a


def masked_allreduce(views: Sequence[torch.Tensor], contrib: Sequence[bool],
                     divisor: float = 0.0) -> None:
    """rcv_masked_allreduce (same device) or the multi-device variant."""
    lib = load()
    n = len(views)
    if n == 0:
        return
    mask = 0
    for i, c in enumerate(contrib):
        if c:
            mask |= 1 << i
    try:
        key = (mask, tuple([(v.data_ptr(), v.numel(), v.dtype, v.stride(0), v.is_cuda)
                            for v in views]))
    except (AttributeError, RuntimeError, IndexError):
        key = None  # not tensors / not 1-D: the full checks raise the right error
    a = _ar_cache.get(key) if key is not None else None
    if a is None:
        a = _prepare_allreduce(views, n, mask)
        if key is not None:
            _ar_cache[key] = a
            if len(_ar_cache) > 256:
                _ar_cache.popitem(last=False)
    if not a.multi:
        _check(lib.rcv_masked_allreduce(a.ptrs, n, mask, a.code, a.numel, float(divisor),
                                        raw_stream(a.first_dev)))
        return
    streams = (ctypes.c_void_p * len(a.devs))(*[raw_stream(d) for d in a.devs])
    _check(lib.rcv_masked_allreduce_multidev(a.ptrs, n, mask, a.code, a.numel, float(divisor),
                                             len(a.devs), a.dev_arr, streams))


_peer_done: set = set()


def enable_peer_access(devices: Sequence[int]) -> None:
    key = tuple(sorted(set(devices)))
    if len(key) < 2 or key in _peer_done:
        return
    arr = (ctypes.c_int * len(key))(*key)
    _check(load().rcv_enable_peer_access(len(key), arr))
    _peer_done.add(key)


def accumulate(acc: torch.Tensor, grad: torch.Tensor, first: bool = False) -> None:
    require_cuda(acc, "accumulator")
    require_cuda(grad, "gradient")
    if acc.numel() != grad.numel():
        raise ValueError("accumulator and gradient differ in length")
    _check(load().rcv_accumulate(acc.data_ptr(), grad.data_ptr(),
                                 dtype_code(acc), dtype_code(grad),
                                 acc.numel(), int(first), stream_of(acc)))


KACC_MAX_SEGS, KACC_MAX_DEPTH = 256, 8


def kacc_push(grads: Sequence[torch.Tensor], stack: Sequence[torch.Tensor],
              out: torch.Tensor) -> None:
    """rcv_kacc_push: out = stack[0] + (... + (stack[-1] + flat(grads))),
    where flat(grads) is the concatenation of the per-parameter gradient
    tensors in order (read in place, no flattening copy).  out may be
    stack[0] (in-place merge) or a fresh buffer (empty stack)."""
    require_cuda(out, "K-ACC output")
    n = len(grads)
    if n == 0 or n > KACC_MAX_SEGS:
        raise ValueError("K-ACC takes 1..%d gradient segments, got %d" % (KACC_MAX_SEGS, n))
    if len(stack) > KACC_MAX_DEPTH:
        raise ValueError("K-ACC carry chain longer than %d" % KACC_MAX_DEPTH)
    dt = dtype_code(grads[0])
    ptrs = (ctypes.c_void_p * n)()
    offs = (ctypes.c_uint64 * n)()
    lens = (ctypes.c_uint64 * n)()
    pos = 0
    for i, g in enumerate(grads):
        if not g.is_cuda or not g.is_contiguous() or dtype_code(g) != dt:
            raise ValueError("K-ACC gradient segment %d must be a contiguous CUDA tensor of one "
                             "dtype" % i)
        ptrs[i], offs[i], lens[i] = g.data_ptr(), pos, g.numel()
        pos += g.numel()
    for s in stack:
        require_cuda(s, "K-ACC stack entry")
    st = _ptrs(stack)
    _check(load().rcv_kacc_push(ptrs, offs, lens, n, dt, st, len(stack), out.data_ptr(),
                                out.numel(), stream_of(out)))


def tree_program(blocks: Sequence[tuple], n_leaves: int):
    """(lo, level) blocks in ascending lo -> (ops bytes, max depth)."""
    n = len(blocks)
    lo = (ctypes.c_uint32 * max(1, n))(*[b[0] for b in blocks])
    lev = (ctypes.c_uint32 * max(1, n))(*[b[1] for b in blocks])
    ops = (ctypes.c_uint8 * max(1, n))()
    depth = ctypes.c_int(0)
    _check(load().rcv_tree_program(lo, lev, n, n_leaves, ops,
                                   ctypes.byref(depth)))
    return list(ops)[:n], depth.value


def tree_commit(blocks: Sequence[tuple], n_leaves: int,
                outputs: Sequence[torch.Tensor], divisor: float,
                variant: int = VARIANT_AUTO) -> None:
    """blocks: sequence of (tensor, lo, level), ascending lo."""
    if not outputs:
        return
    acc = outputs[0]
    arr = (_Block * max(1, len(blocks)))()
    for i, (t, lo, level) in enumerate(blocks):
        require_cuda(t, "block partial")
        if t.numel() != acc.numel():
            raise ValueError("block partial length differs from the output")
        arr[i] = _Block(t.data_ptr(), lo, level, dtype_code(t))
    for o in outputs:
        require_cuda(o, "commit output")
    _check(load().rcv_tree_commit(arr, len(blocks), n_leaves, len(outputs),
                                  _ptrs(outputs), dtype_code(acc),
                                  acc.numel(), float(divisor), variant,
                                  stream_of(acc)))


def copy_(dst: torch.Tensor, src: torch.Tensor) -> None:
    require_cuda(dst, "copy destination")
    require_cuda(src, "copy source")
    if dst.numel() != src.numel() or dst.dtype != src.dtype:
        raise ValueError("copy operands differ")
    _check(load().rcv_copy(dst.data_ptr(), src.data_ptr(),
                           dst.numel() * dst.element_size(), stream_of(dst)))


def zero_(dst: torch.Tensor) -> None:
    require_cuda(dst, "zero target")
    _check(load().rcv_zero(dst.data_ptr(), dst.numel() * dst.element_size(),
                           stream_of(dst)))


def count_differences(a: torch.Tensor, b: torch.Tensor,
                      counter: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Device uint64 (as int64 tensor) count of differing 32-bit words."""
    require_cuda(a)
    require_cuda(b)
    if a.numel() * a.element_size() != b.numel() * b.element_size():
        return torch.ones((), dtype=torch.int64, device=a.device)
    if counter is None:
        counter = torch.zeros((), dtype=torch.int64, device=a.device)
    _check(load().rcv_compare(a.data_ptr(), b.data_ptr(),
                              a.numel() * a.element_size(),
                              counter.data_ptr(), stream_of(a)))
    return counter


def sgd_commit(params: torch.Tensor, flat: torch.Tensor, b: float,
               lr: float) -> None:
    require_cuda(params, "params")
    require_cuda(flat, "flat gradient")
    if params.dtype != flat.dtype or params.numel() != flat.numel():
        raise ValueError("params/flat mismatch")
    _check(load().rcv_sgd_commit(params.data_ptr(), flat.data_ptr(),
                                 dtype_code(params), params.numel(),
                                 float(b), float(lr), stream_of(params)))


def unit_lanes(out: torch.Tensor, base: int, scale: float = 1.0,
               shift: float = 0.0, floor7: bool = False) -> None:
    require_cuda(out, "lanes")
    if out.dtype != torch.float64:
        raise TypeError("lanes are float64")
    _check(load().rcv_unit_lanes(out.data_ptr(), base & ((1 << 64) - 1),
                                 out.numel(), float(scale), float(shift),
                                 int(floor7), stream_of(out)))


def toy_grad(linear: bool, params: torch.Tensor, lanes: torch.Tensor,
             wstar: Optional[torch.Tensor], grad: torch.Tensor,
             scal: torch.Tensor) -> None:
    for t in (params, lanes, scal) + ((grad,) if grad is not None else ()):
        require_cuda(t)
    dim = params.numel()
    _check(load().rcv_toy_grad(int(linear), params.data_ptr(),
                               lanes.data_ptr(),
                               wstar.data_ptr() if wstar is not None else None,
                               dim, grad.data_ptr() if grad is not None else None,
                               scal.data_ptr(),
                               stream_of(scal)))


# ---- multi-process helpers -------------------------------------------------

def ipc_export(t: torch.Tensor):
    """(64-byte handle, offset) of the allocation holding t."""
    require_cuda(t.view(-1) if t.dim() != 1 else t, "shared buffer")
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_size_t(0)
    _check(load().rcv_ipc_export(t.data_ptr(), h, ctypes.byref(off)))
    return h.raw, off.value


def ipc_import(handle: bytes, offset: int) -> int:
    ptr = ctypes.c_void_p(0)
    buf = ctypes.create_string_buffer(handle, 64)
    _check(load().rcv_ipc_import(buf, offset, ctypes.byref(ptr)))
    return ptr.value


def barrier(local_flags: torch.Tensor, peer_flag_ptrs: Sequence[int], me: int,
            live_mask: int, value: int, timeout_ns: int,
            status: torch.Tensor) -> None:
    n = len(peer_flag_ptrs)
    arr = (ctypes.c_void_p * n)(*peer_flag_ptrs)
    _check(load().rcv_barrier(local_flags.data_ptr(), arr, n, me, live_mask,
                              value, timeout_ns, status.data_ptr(),
                              stream_of(local_flags)))


class TreePlan:
    """Prebuilt pointer arrays for repeated rcv_tree_commit_at calls: one
    plan per (cover, outputs), then one cheap call per bucket or slice.
    blocks = [(base_ptr, lo, level, dtype)], ascending lo; outs = [base_ptr]."""

    def __init__(self, blocks: Sequence[tuple], n_leaves: int,
                 outs: Sequence[int], acc_dtype: int, divisor: float,
                 variant: int = VARIANT_AUTO):
        self.n = len(blocks)
        self.arr = (_Block * max(1, self.n))()
        for i, (ptr, lo, level, dt) in enumerate(blocks):
            self.arr[i] = _Block(ptr, lo, level, dt)
        self.n_out = len(outs)
        self.outs = (ctypes.c_void_p * max(1, self.n_out))(*outs)
        self.n_leaves = n_leaves
        self.acc = acc_dtype
        self.divisor = float(divisor)
        self.variant = variant
        self.fn = load().rcv_tree_commit_at

    def run(self, in_offset: int, out_offset: int, numel: int, stream: int) -> None:
        if numel == 0 or self.n_out == 0:
            return
        _check(self.fn(self.arr, self.n, self.n_leaves, self.n_out, self.outs,
                       self.acc, in_offset, out_offset, numel, self.divisor,
                       self.variant, stream))


KIND_NAMES = ("prereduce", "barrier", "broadcast", "combine")


def pool_sets() -> int:
    """Partial-pool sets the native runtime rotates through (rcv_pool_sets)."""
    return int(load().rcv_pool_sets())


class BucketRuntime:
    """The native per-bucket runtime of one rank (rcv_ctx) and its current
    plan (rcv_plan)."""

    def __init__(self, n_ranks: int, me: int, flags: torch.Tensor,
                 peer_flag_ptrs: Sequence[int], status: torch.Tensor,
                 timeout_ns: int):
        lib = load()
        arr = (ctypes.c_void_p * n_ranks)(*peer_flag_ptrs)
        h = ctypes.c_void_p(0)
        _check(lib.rcv_ctx_create(n_ranks, me, flags.data_ptr(), arr,
                                  status.data_ptr(), timeout_ns, ctypes.byref(h)))
        self.ctx = h
        self.plan = None
        self._keep = None
        # native plans by leaf layout: a failure-free step reuses the plan of
        # the step before it instead of rebuilding it (host time per step)
        self._cache: "OrderedDict" = OrderedDict()
        self.cache_size = 8

    def set_plan(self, desc: "PlanDesc", keep, key=None) -> None:
        h = ctypes.c_void_p(0)
        _check(load().rcv_plan_create(self.ctx, ctypes.byref(desc), ctypes.byref(h)))
        if key is None:
            if self.plan is not None and not any(v[0] is self.plan for v in self._cache.values()):
                load().rcv_plan_destroy(self.plan)
            self.plan, self._keep = h, keep
            return
        self._cache[key] = (h, keep)
        self.plan, self._keep = h, keep
        while len(self._cache) > self.cache_size:
            _, (old, _) = self._cache.popitem(last=False)
            load().rcv_plan_destroy(old)

    def use_cached(self, key) -> bool:
        """Make the cached plan of `key` current; False when there is none."""
        hit = self._cache.get(key)
        if hit is None:
            return False
        self._cache.move_to_end(key)
        self.plan, self._keep = hit
        return True

    def bucket(self, lo: int, n: int, stream: int) -> None:
        _check(load().rcv_plan_bucket(self.plan, lo, n, stream))

    def finish(self, live_mask: int, participate: bool, stream: int) -> None:
        _check(load().rcv_ctx_finish(self.ctx, live_mask, int(participate), stream))

    def poll(self, live_mask: int, participate: bool, stream: int) -> None:
        _check(load().rcv_ctx_poll(self.ctx, live_mask, int(participate), stream))

    def set_timing(self, on: bool) -> None:
        _check(load().rcv_ctx_set_timing(self.ctx, int(on)))

    def set_liveness(self, lv: Optional["Liveness"]) -> None:
        _check(load().rcv_ctx_set_liveness(self.ctx, lv.device_word if lv else None))

    def timings(self, max_n: int = 1 << 16):
        kind = (ctypes.c_int * max_n)()
        ms = (ctypes.c_float * max_n)()
        by = (ctypes.c_double * max_n)()
        ni = (ctypes.c_double * max_n)()
        no = (ctypes.c_double * max_n)()
        cnt = ctypes.c_int(0)
        _check(load().rcv_ctx_timing(self.ctx, max_n, kind, ms, by, ni, no, ctypes.byref(cnt)))
        return [(KIND_NAMES[kind[i]], ms[i], by[i], ni[i], no[i]) for i in range(cnt.value)]

    def close(self) -> None:
        lib = load()
        for h, _ in self._cache.values():
            if h is not self.plan:
                lib.rcv_plan_destroy(h)
        self._cache.clear()
        if self.plan is not None:
            lib.rcv_plan_destroy(self.plan)
            self.plan = None
        if self.ctx:
            lib.rcv_ctx_destroy(self.ctx)
            self.ctx = None


def launch_count() -> int:
    """Kernels launched by librcv.so so far in this process."""
    return int(load().rcv_launch_count())


# ---- VMM shareable memory (real-kill mode) -----------------------------------

def vmm_alloc(nbytes: int):
    """(device ptr, mapped size, exported POSIX fd) on the current GPU."""
    ptr, size, fd = ctypes.c_void_p(0), ctypes.c_size_t(0), ctypes.c_int(-1)
    _check(load().rcv_vmm_alloc(nbytes, ctypes.byref(ptr), ctypes.byref(size), ctypes.byref(fd)))
    return ptr.value, size.value, fd.value


def vmm_import(fd: int, size: int, owner_device: int) -> int:
    ptr = ctypes.c_void_p(0)
    _check(load().rcv_vmm_import(fd, size, owner_device, ctypes.byref(ptr)))
    return ptr.value


# ---- NVLink SHARP multicast objects (rcv_mc_*) --------------------------------

def mc_supported() -> bool:
    ok = ctypes.c_int(0)
    _check(load().rcv_mc_supported(ctypes.byref(ok)))
    return bool(ok.value)


def mc_granularity(n_dev: int) -> int:
    g = ctypes.c_size_t(0)
    _check(load().rcv_mc_granularity(n_dev, ctypes.byref(g)))
    return g.value


def mc_create(nbytes: int, n_dev: int):
    """(handle, size, exported POSIX fd) of a new multicast object."""
    h, size, fd = ctypes.c_uint64(0), ctypes.c_size_t(0), ctypes.c_int(-1)
    _check(load().rcv_mc_create(nbytes, n_dev, ctypes.byref(h), ctypes.byref(size),
                                ctypes.byref(fd)))
    return h.value, size.value, fd.value


def mc_import(fd: int) -> int:
    h = ctypes.c_uint64(0)
    _check(load().rcv_mc_import(fd, ctypes.byref(h)))
    return h.value


def mc_add_device(handle: int) -> None:
    _check(load().rcv_mc_add_device(handle))


def mc_bind(handle: int, ptr: int, nbytes: int) -> None:
    _check(load().rcv_mc_bind(handle, ptr, nbytes))


def mc_map(handle: int, size: int) -> int:
    ptr = ctypes.c_void_p(0)
    _check(load().rcv_mc_map(handle, size, ctypes.byref(ptr)))
    return ptr.value


def mc_release(handle: int, ptr: int, size: int) -> None:
    _check(load().rcv_mc_release(handle, ptr, size))


class _CudaArray:
    """__cuda_array_interface__ over raw device memory (for torch.as_tensor)."""

    def __init__(self, ptr: int, numel: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (numel,), "typestr": typestr,
                                         "data": (ptr, False), "version": 2,
                                         "strides": None}


def tensor_at(ptr: int, numel: int, dtype: torch.dtype, device) -> torch.Tensor:
    """A torch view of `numel` elements at device address ptr (no copy)."""
    typestr = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8",
               torch.int32: "<i4"}[dtype]
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, numel, typestr), device=device)


class Liveness:
    """rcv_liveness: node-local heartbeat and failed-set agreement of one
    rank (include/rcv.h).  Every rank of the group must create it with the
    same `name` before any of them relies on it (a barrier after create)."""

    def __init__(self, name: str, rank: int, world: int, period_s: float = 1e-3,
                 deadline_s: float = 10e-3):
        h = ctypes.c_void_p(0)
        _check(load().rcv_liveness_create(name.encode(), rank, world, int(period_s * 1e9),
                                          int(deadline_s * 1e9), ctypes.byref(h)))
        self.h, self.rank, self.world, self.name = h, rank, world, name
        dp, now = ctypes.c_void_p(0), ctypes.c_uint32(0)
        _check(load().rcv_liveness_dead_word(self.h, ctypes.byref(dp), ctypes.byref(now)))
        self.device_word = dp.value

    def dead(self) -> int:
        now = ctypes.c_uint32(0)
        _check(load().rcv_liveness_dead_word(self.h, None, ctypes.byref(now)))
        return now.value

    def decide(self, seq: int):
        """(agreed dead mask, CLOCK_MONOTONIC ns it was decided) of poll seq."""
        m, t = ctypes.c_uint32(0), ctypes.c_uint64(0)
        _check(load().rcv_liveness_decide(self.h, seq, ctypes.byref(m), ctypes.byref(t)))
        return m.value, t.value

    def stats(self, rank: int) -> dict:
        v = [ctypes.c_uint64(0) for _ in range(4)]
        _check(load().rcv_liveness_stats(self.h, rank, *[ctypes.byref(x) for x in v]))
        return dict(beat_ns=v[0].value, dead_ns=v[1].value, kill_ns=v[2].value, now_ns=v[3].value)

    def note_kill(self) -> None:
        _check(load().rcv_liveness_note_kill(self.h))

    def close(self, unlink: bool = False) -> None:
        if self.h:
            load().rcv_liveness_destroy(self.h, int(unlink))
            self.h = None
