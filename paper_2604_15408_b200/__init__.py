"""Thin Python binding of libragged.so (include/ragged.h) -- argument
marshalling only.  Every step of the pack-attend-unpack path runs in the CUDA
kernels of csrc/; there is no CPU or PyTorch fallback: the first call raises
ImportError if the shared library is missing (the package itself imports
without it so that `python -m paper_2604_15408_b200.build` can build it), and
every call raises RaggedError on a non-OK status.  PyTorch is used only for device memory and streams.

Names follow the C ABI: scan, pack, attn, unpack, pack_attend_unpack, Graph,
empty_launch (ragged_scan, ragged_pack, ...).  Citations: PAPER.md lines
P:266-277 (packing), P:286-334 (Alg. 1, grid), BASELINE.json north_star.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# RAGGED_LIB selects another build of the same ABI (e.g. the timeline debug
# build libragged_tl.so used by scripts/timeline.py); default libragged.so.
LIB_PATH = os.environ.get("RAGGED_LIB") or os.path.join(_PKG, "libragged.so")

BF16, FP16 = 0, 1
ENGINE_AUTO, ENGINE_MMA_SYNC, ENGINE_TCGEN05, ENGINE_TCGEN05_WS = 0, 1, 2, 3
OK, EINVAL, ENOTSUP, EALIGN, ECUDA = 0, 1, 2, 3, 4
_DTYPE = {torch.bfloat16: BF16, torch.float16: FP16}


class RaggedError(RuntimeError):
    def __init__(self, status: int, fn: str):
        self.status = status
        super().__init__(f"{fn}: {status_str(status)}: {last_error()}")


class Problem(ctypes.Structure):
    """ragged_problem: B images, N padded tokens (incl. CLS), H heads, d = 64,
    dtype, engine, ld = token stride of padded q/k/v in elements, n_hint =
    expected kept tokens per image (0 = unknown; performance only)."""
    _fields_ = [("B", ctypes.c_int32), ("N", ctypes.c_int32), ("H", ctypes.c_int32),
                ("d", ctypes.c_int32), ("dtype", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("ld", ctypes.c_int64), ("n_hint", ctypes.c_int32)]


MAX_PEERS = 8


class Gather(ctypes.Structure):
    """ragged_gather (include/ragged_dist.h): per-rank destinations of this
    rank's output shard (device pointers, peer-mapped for other ranks), the
    ranks' signal arrays and this rank's barrier state."""
    _fields_ = [("world", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("out", ctypes.c_void_p * MAX_PEERS), ("cls", ctypes.c_void_p * MAX_PEERS),
                ("signal", ctypes.c_void_p * MAX_PEERS), ("state", ctypes.c_void_p)]


def _addr(x) -> int | None:
    """A device address: a tensor's data_ptr(), a raw int (e.g. a peer pointer
    from torch symmetric memory), or None."""
    if x is None:
        return None
    return x.data_ptr() if hasattr(x, "data_ptr") else int(x)


def gather_desc(world: int, rank: int, out=None, cls=None, signal=None, state=None) -> Gather:
    """Build a ragged_gather from per-rank lists (length world; entries are
    tensors, ints or None)."""
    g = Gather()
    g.world, g.rank = world, rank
    for name, lst in (("out", out), ("cls", cls), ("signal", signal)):
        if lst is None:
            continue
        if len(lst) != world:
            raise ValueError(f"{name} must have one entry per rank")
        arr = getattr(g, name)
        for r, x in enumerate(lst):
            arr[r] = _addr(x)
    g.state = _addr(state)
    return g


EPI_NONE, EPI_GELU, EPI_RESIDUAL = 0, 1, 2
VIT_PARAMS = ("ln1_w", "ln1_b", "w_qkv", "b_qkv", "w_proj", "b_proj",
              "ln2_w", "ln2_b", "w_fc1", "b_fc1", "w_fc2", "b_fc2")


class VitWeights(ctypes.Structure):
    """ragged_vit_weights (include/ragged_block.h)."""
    _fields_ = [(n, ctypes.c_void_p) for n in VIT_PARAMS] + [("mlp", ctypes.c_int32)]


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2604_15408_b200.build` "
                          "(there is no fallback path)")
    lib = ctypes.CDLL(LIB_PATH)
    P, V, I32, I64 = ctypes.POINTER(Problem), ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    sigs = {
        "ragged_scan": [P, V, V, V, V, V],
        "ragged_pack": [P, V, V, V, V, V, V, V, V, V, V, V],
        "ragged_attn": [P, V, V, V, V, V, V],
        "ragged_unpack": [P, V, V, V, V],
        "ragged_attn_fp8": [P, V, V, V, ctypes.c_float, ctypes.c_float, ctypes.c_float, V, V, V],
        "ragged_pack_attend_unpack": [P, V, V, V, V, V, V, V],
        "ragged_pack_attend_unpack_host": [P, V, V, V, V, V, V, V],
        "ragged_graph_create": [P, V, V, V, V, V, V, ctypes.POINTER(V)],
        "ragged_graph_launch": [V, V],
        "ragged_empty_launch": [I32, I32, V],
        "ragged_keep_topk_l2": [P, V, I32, V, V],
        "ragged_keep_evit": [P, V, V, V, I32, V, V],
        "ragged_prune_l2_pack_attend_unpack": [P, V, I64, I32, V, V, V, V, V, V, V],
        "ragged_validate_cu_seqlens": [ctypes.POINTER(I32), I32, I64],
        "ragged_pack_attend_unpack_gather": [P, V, V, V, V, V, ctypes.POINTER(Gather), V],
        "ragged_attn_gather": [P, V, V, V, V, ctypes.POINTER(Gather), V],
        "ragged_layer_norm": [I32, I32, I32, V, I64, V, V, ctypes.c_float, V, I64, V, V],
        "ragged_linear": [I32, I32, I32, I32, V, I64, V, V, I32, V, I64, V, I64, V, V],
        "ragged_vit_block": [P, V, V, ctypes.POINTER(VitWeights), V, I64, V],
        "ragged_pack_rows": [P, V, V, V, V, V, V, V],
        "ragged_dist_nccl_available": [],
        "ragged_dist_nccl_unique_id": [V],
        "ragged_dist_nccl_init": [V, I32, I32, ctypes.POINTER(V)],
        "ragged_dist_nccl_init_all": [I32, V, V],
        "ragged_dist_pack_attend_unpack_allgather": [P, V, V, V, V, V, V, V, V, V],
        "ragged_dist_cls_allgather": [P, V, V, V, V, V, V, V, V, V],
        "ragged_cls_rows": [P, V, V, V, V],
        "ragged_vit_pipeline_graph_create": [P, V, V, ctypes.POINTER(VitWeights), I32, V, I64, ctypes.POINTER(V)],
    }
    for name, args in sigs.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int32
    lib.ragged_vit_block_workspace.argtypes = [P, I32]
    lib.ragged_vit_block_workspace.restype = ctypes.c_int64
    lib.ragged_graph_destroy.argtypes = [V]
    lib.ragged_graph_destroy.restype = None
    lib.ragged_dist_nccl_destroy.argtypes = [V]
    lib.ragged_dist_nccl_destroy.restype = None
    lib.ragged_status_str.argtypes = [ctypes.c_int32]
    lib.ragged_status_str.restype = ctypes.c_char_p
    lib.ragged_last_error.argtypes = []
    lib.ragged_last_error.restype = ctypes.c_char_p
    lib.ragged_build_info.argtypes = []
    lib.ragged_build_info.restype = ctypes.c_char_p
    return lib


_lib = None

EXPORTS = ("ragged_scan", "ragged_pack", "ragged_attn", "ragged_unpack", "ragged_pack_attend_unpack",
           "ragged_pack_attend_unpack_host", "ragged_attn_fp8",
           "ragged_graph_create", "ragged_graph_launch", "ragged_graph_destroy", "ragged_empty_launch",
           "ragged_validate_cu_seqlens", "ragged_status_str", "ragged_last_error", "ragged_build_info",
           "ragged_keep_topk_l2", "ragged_keep_evit", "ragged_prune_l2_pack_attend_unpack", "ragged_pack_attend_unpack_gather", "ragged_attn_gather",
           "ragged_layer_norm", "ragged_linear", "ragged_vit_block_workspace", "ragged_vit_block",
           "ragged_pack_rows", "ragged_cls_rows", "ragged_dist_nccl_available", "ragged_dist_nccl_unique_id",
           "ragged_dist_nccl_init", "ragged_dist_nccl_init_all", "ragged_dist_nccl_destroy",
           "ragged_dist_pack_attend_unpack_allgather", "ragged_dist_cls_allgather",
           "ragged_vit_pipeline_graph_create")


def lib() -> ctypes.CDLL:
    """The loaded libragged.so (loaded on first use; raises if it is missing)."""
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def status_str(s: int) -> str:
    return lib().ragged_status_str(s).decode()


def last_error() -> str:
    return lib().ragged_last_error().decode()


def build_info() -> str:
    return lib().ragged_build_info().decode()


def _check(status: int, fn: str) -> None:
    if status != OK:
        raise RaggedError(status, fn)


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def _stream(stream) -> int | None:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def problem(B: int, N: int, H: int, d: int = 64, dtype=torch.bfloat16, ld: int | None = None,
            engine: int = ENGINE_AUTO, n_hint: int = 0) -> Problem:
    dt = _DTYPE[dtype] if isinstance(dtype, torch.dtype) else int(dtype)
    return Problem(B, N, H, d, dt, engine, H * d if ld is None else ld, n_hint)


def _padded_problem(q, k, v, engine, n_hint=0):
    """Problem for padded q/k/v [B, N, H, d] views sharing one token stride."""
    if q.dim() != 4:
        raise ValueError("q/k/v must be [B, N, H, d]")
    B, N, H, d = q.shape
    for t in (k, v):
        if t.shape != q.shape or t.stride() != q.stride() or t.dtype != q.dtype:
            raise ValueError("q, k, v must share shape, strides and dtype")
    if q.stride(3) != 1 or q.stride(2) != d or q.stride(0) != N * q.stride(1):
        raise ValueError("q/k/v must be token-major [B, N, H, d] with unit head-dim stride")
    if q.dtype not in _DTYPE:
        raise ValueError("dtype must be bf16 or fp16")
    return problem(B, N, H, d, q.dtype, q.stride(1), engine, n_hint)


def _keep_u8(keep, B: int | None = None, N: int | None = None, device=None):
    if keep.dtype == torch.bool:
        keep = keep.view(torch.uint8)
    if keep.dtype != torch.uint8 or not keep.is_contiguous() or keep.dim() != 2:
        raise ValueError("keep must be a contiguous uint8/bool [B, N] tensor")
    if B is not None and tuple(keep.shape) != (B, N):
        raise ValueError(f"keep must be [B, N] = [{B}, {N}], got {list(keep.shape)}")
    if device is not None and keep.device != device:
        raise ValueError(f"keep is on {keep.device}, expected {device}")
    return keep


def _require(t, name: str, dtype, device, numel: int | None = None, shape=None):
    """The C ABI cannot see buffer sizes: check a caller buffer before its
    pointer crosses the boundary (dtype, device, contiguity, size)."""
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {list(shape)}, got {list(t.shape)}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"{name} holds {t.numel()} elements, needs at least {numel}")
    return t


def scan(keep, cu=None, dst=None, src=None, stream=None):
    """a1: keep [B, N] -> (cu [B+1], dst [B*N], src [B*N] capacity)."""
    keep = _keep_u8(keep)
    B, N = keep.shape
    dev = keep.device
    cu = torch.empty(B + 1, dtype=torch.int32, device=dev) if cu is None else cu
    dst = torch.empty(B * N, dtype=torch.int32, device=dev) if dst is None else dst
    src = torch.empty(B * N, dtype=torch.int32, device=dev) if src is None else src
    _require(cu, "cu", torch.int32, dev, B + 1)
    _require(dst, "dst", torch.int32, dev, B * N)
    _require(src, "src", torch.int32, dev, B * N)
    p = problem(B, N, 1)
    _check(lib().ragged_scan(ctypes.byref(p), keep.data_ptr(), cu.data_ptr(), dst.data_ptr(),
                            src.data_ptr(), _stream(stream)), "ragged_scan")
    return cu, dst, src


def pack(q, k, v, keep, out=None, stream=None, engine=ENGINE_AUTO):
    """a1 + a2: returns (qp, kp, vp, cu, dst, src); packed buffers
    have capacity B*N rows, rows [0, cu[B]) valid."""
    p = _padded_problem(q, k, v, engine)
    B, N, H, d = q.shape
    keep = _keep_u8(keep, B, N, q.device)
    if out is None:
        mk = lambda: torch.empty(B * N, H, d, dtype=q.dtype, device=q.device)  # noqa: E731
        qp, kp, vp = mk(), mk(), mk()
        cu = torch.empty(B + 1, dtype=torch.int32, device=q.device)
        dst = torch.empty(B * N, dtype=torch.int32, device=q.device)
        src = torch.empty(B * N, dtype=torch.int32, device=q.device)
    else:
        qp, kp, vp, cu, dst, src = out
        for t, nm in ((qp, "qp"), (kp, "kp"), (vp, "vp")):
            _require(t, nm, q.dtype, q.device, B * N * H * d)
        for t, nm in ((cu, "cu"), (dst, "dst"), (src, "src")):
            _require(t, nm, torch.int32, q.device, B + 1 if nm == "cu" else B * N)
    _check(lib().ragged_pack(ctypes.byref(p), keep.data_ptr(), q.data_ptr(), k.data_ptr(), v.data_ptr(),
                            cu.data_ptr(), dst.data_ptr(), src.data_ptr(), qp.data_ptr(), kp.data_ptr(),
                            vp.data_ptr(), _stream(stream)), "ragged_pack")
    return qp, kp, vp, cu, dst, src


def _packed_ld(qp, kp, vp) -> int:
    """Row stride of packed q/k/v [cap, H, d] views: contiguous buffers (H*d)
    or slices of one packed qkv buffer [cap, 3, H, d] (3*H*d)."""
    cap, H, d = qp.shape
    for t in (qp, kp, vp):
        if t.shape != qp.shape or t.dtype != qp.dtype or t.stride() != qp.stride():
            raise ValueError("packed q/k/v must share shape, dtype and strides")
    if qp.stride(2) != 1 or qp.stride(1) != d:
        raise ValueError("packed q/k/v must be [cap, H, d] with contiguous heads")
    return qp.stride(0)


def attn(qp, kp, vp, cu, N: int, op=None, stream=None, engine=ENGINE_AUTO, n_hint=0):
    """a3 (Alg. 1): packed [cap, H, d] + cu [B+1] -> packed O.
    n_hint: expected kept tokens per image (performance only)."""
    cap, H, d = qp.shape
    ld = _packed_ld(qp, kp, vp)
    _require(cu, "cu", torch.int32, qp.device)
    B = cu.numel() - 1
    if cap < B * N:
        raise ValueError(f"packed buffers hold {cap} rows, need capacity B*N = {B * N}")
    op = torch.empty(cap, H, d, dtype=qp.dtype, device=qp.device) if op is None else op
    _require(op, "op", qp.dtype, qp.device, shape=qp.shape)
    p = problem(B, N, H, d, qp.dtype, ld, engine, n_hint)
    _check(lib().ragged_attn(ctypes.byref(p), qp.data_ptr(), kp.data_ptr(), vp.data_ptr(), cu.data_ptr(),
                            op.data_ptr(), _stream(stream)), "ragged_attn")
    return op


def attn_fp8(qp, kp, vp, cu, N: int, descale=(1.0, 1.0, 1.0), out_dtype=torch.bfloat16, op=None,
             stream=None):
    """NEXT row N4: ragged_attn over packed FP8 E4M3 q/k/v ([cap, H, d],
    torch.float8_e4m3fn or uint8 bytes) with per-tensor descale factors
    (descale_q, descale_k, descale_v); output in out_dtype (bf16 / fp16)."""
    if qp.dim() != 3:
        raise ValueError("qp/kp/vp must be packed [cap, H, d]")
    cap, H, d = qp.shape
    for t in (qp, kp, vp):
        if t.dtype not in (torch.float8_e4m3fn, torch.uint8) or t.shape != qp.shape or not t.is_contiguous():
            raise ValueError("qp/kp/vp must be contiguous float8_e4m3fn/uint8 [cap, H, d] of one shape")
    if out_dtype not in _DTYPE:
        raise ValueError("out_dtype must be bf16 or fp16")
    _require(cu, "cu", torch.int32, qp.device)
    if cap < (cu.numel() - 1) * N:
        raise ValueError(f"packed buffers hold {cap} rows, need capacity B*N = {(cu.numel() - 1) * N}")
    op = torch.empty(cap, H, d, dtype=out_dtype, device=qp.device) if op is None else op
    _require(op, "op", out_dtype, qp.device, shape=(cap, H, d))
    p = problem(len(cu) - 1, N, H, d, out_dtype, H * d)
    dq, dk, dv = (float(x) for x in descale)
    _check(lib().ragged_attn_fp8(ctypes.byref(p), qp.data_ptr(), kp.data_ptr(), vp.data_ptr(), dq, dk, dv,
                                 cu.data_ptr(), op.data_ptr(), _stream(stream)), "ragged_attn_fp8")
    return op


def unpack(op, dst, B: int, N: int, o=None, stream=None):
    """a4: packed O -> padded [B, N, H, d]; dropped rows +0.0."""
    cap, H, d = op.shape
    if cap < B * N or not op.is_contiguous():
        raise ValueError(f"op must be a contiguous packed buffer of capacity B*N = {B * N} rows")
    _require(dst, "dst", torch.int32, op.device, B * N)
    o = torch.empty(B, N, H, d, dtype=op.dtype, device=op.device) if o is None else o
    _require(o, "o", op.dtype, op.device, shape=(B, N, H, d))
    p = problem(B, N, H, d, op.dtype)
    _check(lib().ragged_unpack(ctypes.byref(p), op.data_ptr(), dst.data_ptr(), o.data_ptr(),
                              _stream(stream)), "ragged_unpack")
    return o


def pack_attend_unpack(q, k, v, keep, o=None, cu=None, want_cu=False, stream=None,
                       engine=ENGINE_AUTO, n_hint=0):
    """a5: the fused single-launch path.  Returns o (and cu if requested).
    n_hint: expected kept tokens per image (performance only)."""
    p = _padded_problem(q, k, v, engine, n_hint)
    B, N, H, d = q.shape
    keep = _keep_u8(keep, B, N, q.device)
    o = torch.empty(B, N, H, d, dtype=q.dtype, device=q.device) if o is None else o
    _require(o, "o", q.dtype, q.device, shape=(B, N, H, d))
    if want_cu and cu is None:
        cu = torch.empty(B + 1, dtype=torch.int32, device=q.device)
    if cu is not None:
        _require(cu, "cu", torch.int32, q.device, B + 1)
    _check(lib().ragged_pack_attend_unpack(ctypes.byref(p), keep.data_ptr(), q.data_ptr(), k.data_ptr(),
                                          v.data_ptr(), o.data_ptr(), _ptr(cu), _stream(stream)),
           "ragged_pack_attend_unpack")
    return (o, cu) if (want_cu or cu is not None) else o


def pack_attend_unpack_host(q, k, v, keep, o, cu=None, stream=None, engine=ENGINE_AUTO):
    """a5 end to end from host memory: q, k, v, keep are PINNED CPU tensors
    (tensor.pin_memory()); the kernel reads the mask and only the kept rows
    over the host link (ragged_pack_attend_unpack_host).  o (and cu) are
    device tensors or pinned CPU tensors.  Returns o."""
    for t in (q, k, v, keep):
        if t.device.type != "cpu" or not t.is_pinned():
            raise ValueError("q, k, v, keep must be pinned CPU tensors")
    p = _padded_problem(q, k, v, engine)
    B, N, H, d = q.shape
    keep = _keep_u8(keep, B, N)
    if o.dtype != q.dtype or tuple(o.shape) != (B, N, H, d) or not o.is_contiguous():
        raise ValueError("o must be a contiguous [B, N, H, d] tensor of q's dtype")
    if o.device.type == "cpu" and not o.is_pinned():
        raise ValueError("a CPU o must be pinned")
    if cu is not None and (cu.dtype != torch.int32 or cu.numel() < B + 1):
        raise ValueError("cu must be int32 with at least B+1 elements")
    _check(lib().ragged_pack_attend_unpack_host(ctypes.byref(p), keep.data_ptr(), q.data_ptr(),
                                               k.data_ptr(), v.data_ptr(), o.data_ptr(), _ptr(cu),
                                               _stream(stream)),
           "ragged_pack_attend_unpack_host")
    return o


def pack_attend_unpack_gather(q, k, v, keep, gather: Gather, cu=None, stream=None,
                              engine=ENGINE_AUTO, n_hint=0):
    """a5 fused with the §8(e) all-gather: this rank's padded O rows (and/or
    CLS rows) are stored into every rank's gathered buffer (ragged_dist.h)."""
    p = _padded_problem(q, k, v, engine, n_hint)
    keep = _keep_u8(keep, q.shape[0], q.shape[1], q.device)
    if cu is not None:
        _require(cu, "cu", torch.int32, q.device, q.shape[0] + 1)
    _check(lib().ragged_pack_attend_unpack_gather(ctypes.byref(p), keep.data_ptr(), q.data_ptr(),
                                                 k.data_ptr(), v.data_ptr(), _ptr(cu),
                                                 ctypes.byref(gather), _stream(stream)),
           "ragged_pack_attend_unpack_gather")


def attn_gather(qp, kp, vp, cu, N: int, gather: Gather, stream=None, engine=ENGINE_AUTO, n_hint=0):
    """a3 with the packed all-gather: rows [cu[b], cu[b+1]) of this rank's
    packed O go to out[r] + row * H * d on every rank r (ragged_dist.h)."""
    cap, H, d = qp.shape
    _require(cu, "cu", torch.int32, qp.device)
    B = cu.numel() - 1
    if cap < B * N:
        raise ValueError(f"packed buffers hold {cap} rows, need capacity B*N = {B * N}")
    p = problem(B, N, H, d, qp.dtype, _packed_ld(qp, kp, vp), engine, n_hint)
    _check(lib().ragged_attn_gather(ctypes.byref(p), qp.data_ptr(), kp.data_ptr(), vp.data_ptr(),
                                   cu.data_ptr(), ctypes.byref(gather), _stream(stream)),
           "ragged_attn_gather")


# ---- §8(e) NCCL exchange inside the library (include/ragged_dist.h) ---------

def nccl_available() -> bool:
    return lib().ragged_dist_nccl_available() == OK


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().ragged_dist_nccl_unique_id(buf), "ragged_dist_nccl_unique_id")
    return bytes(buf)


class NcclComm:
    """One rank's ragged_nccl communicator (ncclCommInitRank on the current
    device) from a 128-byte id shared by the caller (e.g. a torch.distributed
    broadcast of nccl_unique_id() from rank 0)."""

    def __init__(self, uid: bytes, world: int, rank: int):
        if len(uid) != 128:
            raise ValueError("unique id must be 128 bytes")
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        h = ctypes.c_void_p()
        _check(lib().ragged_dist_nccl_init(buf, int(world), int(rank), ctypes.byref(h)), "ragged_dist_nccl_init")
        self._h, self.world, self.rank = h, world, rank

    def close(self):
        if getattr(self, "_h", None):
            lib().ragged_dist_nccl_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pack_attend_unpack_allgather(q, k, v, keep, comm: NcclComm, o_all, cls_all=None, cu=None, stream=None,
                                 engine=ENGINE_AUTO, n_hint=0):
    """This rank's shard -> its slot of o_all [world*B, N, H, d], then the
    library's in-place ncclAllGather (and of cls_all [world*B, H*d] if given)."""
    p = _padded_problem(q, k, v, engine, n_hint)
    B, N, H, d = q.shape
    keep = _keep_u8(keep, B, N, q.device)
    _require(o_all, "o_all", q.dtype, q.device, shape=(comm.world * B, N, H, d))
    if cls_all is not None:
        _require(cls_all, "cls_all", q.dtype, q.device, shape=(comm.world * B, H * d))
    if cu is not None:
        _require(cu, "cu", torch.int32, q.device, B + 1)
    _check(lib().ragged_dist_pack_attend_unpack_allgather(ctypes.byref(p), keep.data_ptr(), q.data_ptr(), k.data_ptr(),
                                                          v.data_ptr(), o_all.data_ptr(), _ptr(cls_all), _ptr(cu),
                                                          comm._h, _stream(stream)),
           "ragged_dist_pack_attend_unpack_allgather")
    return o_all


def cls_allgather(q, k, v, keep, comm: NcclComm, cls_all, o_local=None, cu=None, stream=None, engine=ENGINE_AUTO,
                  n_hint=0):
    p = _padded_problem(q, k, v, engine, n_hint)
    B, N, H, d = q.shape
    keep = _keep_u8(keep, B, N, q.device)
    _require(cls_all, "cls_all", q.dtype, q.device, shape=(comm.world * B, H * d))
    if o_local is not None:
        _require(o_local, "o_local", q.dtype, q.device, shape=(B, N, H, d))
    _check(lib().ragged_dist_cls_allgather(ctypes.byref(p), keep.data_ptr(), q.data_ptr(), k.data_ptr(),
                                           v.data_ptr(), _ptr(o_local), cls_all.data_ptr(), _ptr(cu), comm._h,
                                           _stream(stream)), "ragged_dist_cls_allgather")
    return cls_all


# ---- NEXT row N1: packed ViT block (include/ragged_block.h) -----------------

def _live(live):
    return None if live is None else live.data_ptr()


def layer_norm(x, w, b, eps: float = 1e-6, y=None, live=None, stream=None):
    """y = LN(x) over the last dim of x [rows, D] (row stride x.stride(0));
    live: optional device int32 tensor whose first element is the live row count."""
    rows, D = x.shape
    y = torch.empty(rows, D, dtype=x.dtype, device=x.device) if y is None else y
    _check(lib().ragged_layer_norm(_DTYPE[x.dtype], rows, D, x.data_ptr(), x.stride(0), w.data_ptr(),
                                  b.data_ptr(), eps, y.data_ptr(), y.stride(0), _live(live), _stream(stream)),
           "ragged_layer_norm")
    return y


def linear(a, w, bias=None, epi: int = EPI_NONE, residual=None, out=None, live=None, stream=None):
    """out = epi(a w^T + bias) on tcgen05: a [rows, K], w [N, K] (torch Linear layout)."""
    rows, K = a.shape
    N = w.shape[0]
    if w.shape[1] != K or w.stride(1) != 1 or w.stride(0) != K or a.stride(1) != 1:
        raise ValueError("a must be [rows, K] with unit column stride and w contiguous [N, K]")
    out = torch.empty(rows, N, dtype=a.dtype, device=a.device) if out is None else out
    _check(lib().ragged_linear(_DTYPE[a.dtype], rows, N, K, a.data_ptr(), a.stride(0), w.data_ptr(),
                              _ptr(bias), epi, _ptr(residual), 0 if residual is None else residual.stride(0),
                              out.data_ptr(), out.stride(0), _live(live), _stream(stream)), "ragged_linear")
    return out


def vit_weights(params: dict) -> VitWeights:
    """ragged_vit_weights from a dict of device tensors (names VIT_PARAMS)."""
    w = VitWeights()
    for n in VIT_PARAMS:
        setattr(w, n, params[n].data_ptr())
    w.mlp = params["w_fc1"].shape[0]
    return w


class VitBlock:
    """One packed pre-norm ViT block (ragged_vit_block) with its weights and
    a workspace sized for B*N capacity rows."""

    def __init__(self, params: dict, B: int, N: int, H: int, dtype=torch.bfloat16, n_hint: int = 0):
        """n_hint: expected kept tokens per image (performance only)."""
        self.params = params
        self.w = vit_weights(params)
        self.p = problem(B, N, H, 64, dtype, n_hint=n_hint)
        nbytes = lib().ragged_vit_block_workspace(ctypes.byref(self.p), self.w.mlp)
        if nbytes < 0:
            raise ValueError("invalid block problem")
        dev = params["w_qkv"].device
        self.ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=dev)

    def __call__(self, x, cu, stream=None):
        """In place on packed rows x [B*N, D]; rows [0, cu[B]) live."""
        _check(lib().ragged_vit_block(ctypes.byref(self.p), x.data_ptr(), cu.data_ptr(), ctypes.byref(self.w),
                                     self.ws.data_ptr(), self.ws.numel(), _stream(stream)), "ragged_vit_block")
        return x


def pack_rows(x, keep, xp=None, cu=None, dst=None, src=None, stream=None):
    """N1 prune point: hidden state x [B, N, D] (D = H*64, unit
    feature stride) -> packed rows xp [B*N, D] + cu [B+1], dst, src."""
    if x.dim() != 3 or x.stride(2) != 1 or x.dtype not in _DTYPE or x.shape[2] % 64 != 0:
        raise ValueError("x must be [B, N, D] bf16/fp16 with D % 64 == 0 and unit feature stride")
    B, N, D = x.shape
    if x.stride(0) != N * x.stride(1):
        raise ValueError("x tokens must be evenly strided")
    keep = _keep_u8(keep, B, N, x.device)
    xp = torch.empty(B * N, D, dtype=x.dtype, device=x.device) if xp is None else xp
    _require(xp, "xp", x.dtype, x.device, numel=B * N * D)
    cu = torch.empty(B + 1, dtype=torch.int32, device=x.device) if cu is None else cu
    dst = torch.empty(B * N, dtype=torch.int32, device=x.device) if dst is None else dst
    src = torch.empty(B * N, dtype=torch.int32, device=x.device) if src is None else src
    for t, nm, n in ((cu, "cu", B + 1), (dst, "dst", B * N), (src, "src", B * N)):
        _require(t, nm, torch.int32, x.device, n)
    p = problem(B, N, D // 64, 64, x.dtype, x.stride(1))
    _check(lib().ragged_pack_rows(ctypes.byref(p), keep.data_ptr(), x.data_ptr(), cu.data_ptr(), dst.data_ptr(),
                                  src.data_ptr(), xp.data_ptr(), _stream(stream)), "ragged_pack_rows")
    return xp, cu, dst, src


def cls_rows(xp, cu, N: int, out=None, stream=None):
    """CLS readout: out[b] = xp[cu[b]] (+0.0 for an empty image)."""
    if xp.dim() != 2 or not xp.is_contiguous() or xp.dtype not in _DTYPE or xp.shape[1] % 64 != 0:
        raise ValueError("xp must be a contiguous [rows, D] bf16/fp16 tensor, D % 64 == 0")
    _require(cu, "cu", torch.int32, xp.device)
    B, D = cu.numel() - 1, xp.shape[1]
    if xp.shape[0] < B * N:
        raise ValueError("xp must hold the B*N-row capacity")
    out = torch.empty(B, D, dtype=xp.dtype, device=xp.device) if out is None else out
    _require(out, "out", xp.dtype, xp.device, shape=(B, D))
    p = problem(B, N, D // 64, 64, xp.dtype)
    _check(lib().ragged_cls_rows(ctypes.byref(p), xp.data_ptr(), cu.data_ptr(), out.data_ptr(), _stream(stream)),
           "ragged_cls_rows")
    return out


class VitPrunedForward:
    """The paper's pruned DeiT forward (§4.4 steps 1-5) as a sequence
    of library calls (plumbing only: every step is a libragged kernel, all
    PDL-chained on one stream, capturable in one CUDA graph):
      1. layers [0, prune_at): dense blocks on all B*N rows (ragged_vit_block with
         the all-kept cu_seqlens b*N -- packed == padded);
      2. Threshold-l2 keep mask of the hidden state (ragged_keep_topk_l2, k kept);
      3. pack the hidden state once (ragged_pack_rows);
      4. layers [prune_at, L): packed blocks (ragged_vit_block on cu);
      5. CLS rows from the packed buffer (ragged_cls_rows).
    Buffers are allocated once; __call__(x) copies the input [B, N, D] into the
    padded buffer and returns the CLS rows [B, D]."""

    def __init__(self, layer_params, B: int, N: int, H: int, k_keep: int, prune_at: int = 4,
                 dtype=torch.bfloat16):
        dev = layer_params[0]["w_qkv"].device
        D = H * 64
        self.B, self.N, self.H, self.D, self.k, self.prune_at = B, N, H, D, int(k_keep), prune_at
        self.dense = [VitBlock(p, B, N, H, dtype, n_hint=N) for p in layer_params[:prune_at]]
        self.packed = [VitBlock(p, B, N, H, dtype, n_hint=min(k_keep, N)) for p in layer_params[prune_at:]]
        self.x = torch.empty(B * N, D, dtype=dtype, device=dev)
        self.xp = torch.empty(B * N, D, dtype=dtype, device=dev)
        self.cu_all = (torch.arange(B + 1, dtype=torch.int32, device=dev) * N).contiguous()
        self.keep = torch.empty(B, N, dtype=torch.uint8, device=dev)
        self.cu = torch.empty(B + 1, dtype=torch.int32, device=dev)
        self.dst = torch.empty(B * N, dtype=torch.int32, device=dev)
        self.src = torch.empty(B * N, dtype=torch.int32, device=dev)
        self.cls = torch.empty(B, D, dtype=dtype, device=dev)

    def run(self, stream=None):
        """Steps 1-5 on the resident input self.x (no host sync)."""
        for blk in self.dense:
            blk(self.x, self.cu_all, stream)
        x3 = self.x.view(self.B, self.N, self.D)
        keep_topk_l2(x3, self.k, keep=self.keep, stream=stream)
        pack_rows(x3, self.keep, xp=self.xp, cu=self.cu, dst=self.dst, src=self.src, stream=stream)
        for blk in self.packed:
            blk(self.xp, self.cu, stream)
        cls_rows(self.xp, self.cu, self.N, out=self.cls, stream=stream)
        return self.cls

    def __call__(self, x, stream=None):
        self.x.view(self.B, self.N, self.D).copy_(x, non_blocking=True)
        return self.run(stream)


class VitPipelineGraph:
    """ragged_vit_pipeline_graph_create: `len(blocks)` packed blocks (VitBlock
    objects sharing B, N, H, dtype) captured as one replayable graph over the
    fixed buffers x [B*N, D] and cu [B+1]; launch() replays every layer."""

    def __init__(self, blocks, x, cu):
        b0 = blocks[0]
        self._refs = (blocks, x, cu)
        arr = (VitWeights * len(blocks))(*[bl.w for bl in blocks])
        self._arr = arr
        h = ctypes.c_void_p()
        _check(lib().ragged_vit_pipeline_graph_create(ctypes.byref(b0.p), x.data_ptr(), cu.data_ptr(), arr,
                                                     len(blocks), b0.ws.data_ptr(), b0.ws.numel(),
                                                     ctypes.byref(h)), "ragged_vit_pipeline_graph_create")
        self._h = h

    def launch(self, stream=None):
        _check(lib().ragged_graph_launch(self._h, _stream(stream)), "ragged_graph_launch")

    def close(self):
        if getattr(self, "_h", None):
            lib().ragged_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Graph:
    """ragged_graph: one captured pack_attend_unpack with fixed pointers."""

    def __init__(self, q, k, v, keep, o, cu=None, engine=ENGINE_AUTO, n_hint=0):
        self._p = _padded_problem(q, k, v, engine, n_hint)
        keep = _keep_u8(keep)
        self._refs = (q, k, v, keep, o, cu)     # keep the buffers alive
        h = ctypes.c_void_p()
        _check(lib().ragged_graph_create(ctypes.byref(self._p), keep.data_ptr(), q.data_ptr(),
                                        k.data_ptr(), v.data_ptr(), o.data_ptr(), _ptr(cu),
                                        ctypes.byref(h)), "ragged_graph_create")
        self._h = h

    def launch(self, stream=None):
        _check(lib().ragged_graph_launch(self._h, _stream(stream)), "ragged_graph_launch")

    def close(self):
        if getattr(self, "_h", None):
            lib().ragged_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def keep_topk_l2(x, k: int, keep=None, stream=None):
    """N2: Threshold-l2 keep mask from hidden states
    x [B, N, D] (token stride x.stride(1)) -> uint8 keep [B, N]."""
    if x.dim() != 3 or x.stride(2) != 1 or x.dtype not in _DTYPE:
        raise ValueError("x must be [B, N, D] bf16/fp16 with unit feature stride")
    B, N, D = x.shape
    if D % 64 != 0 or x.stride(0) != N * x.stride(1):
        raise ValueError("D must be a multiple of 64 and tokens evenly strided")
    keep = torch.empty(B, N, dtype=torch.uint8, device=x.device) if keep is None else keep
    _require(keep, "keep", torch.uint8, x.device, shape=(B, N))
    p = problem(B, N, D // 64, 64, x.dtype, x.stride(1))
    _check(lib().ragged_keep_topk_l2(ctypes.byref(p), x.data_ptr(), int(k), keep.data_ptr(),
                                     _stream(stream)), "ragged_keep_topk_l2")
    return keep


def prune_l2_pack_attend_unpack(x, q, k, v, k_keep: int, o=None, keep=None, cu=None, stream=None,
                                engine=ENGINE_AUTO):
    """N2 fused ahead of the scan: Threshold-l2 keep mask from hidden states
    x [B, N, H*64] computed inside the fused pack-attend-unpack launch.
    Returns o (padded [B, N, H, d]); keep [B, N] / cu [B+1] filled if given."""
    p = _padded_problem(q, k, v, engine)
    B, N, H, d = q.shape
    if x.dim() != 3 or tuple(x.shape) != (B, N, H * d) or x.dtype != q.dtype or x.stride(2) != 1 \
            or x.stride(0) != N * x.stride(1) or x.device != q.device:
        raise ValueError("x must be [B, N, H*d] of q's dtype and device, unit feature stride")
    o = torch.empty(B, N, H, d, dtype=q.dtype, device=q.device) if o is None else o
    _require(o, "o", q.dtype, q.device, shape=(B, N, H, d))
    if keep is not None:
        _require(keep, "keep", torch.uint8, q.device, shape=(B, N))
    if cu is not None:
        _require(cu, "cu", torch.int32, q.device, B + 1)
    _check(lib().ragged_prune_l2_pack_attend_unpack(ctypes.byref(p), x.data_ptr(), x.stride(1), int(k_keep),
                                                    q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(),
                                                    _ptr(keep), _ptr(cu), _stream(stream)),
           "ragged_prune_l2_pack_attend_unpack")
    return o


def keep_evit(q, k, v, k_keep: int, keep=None, stream=None, n_hint=0):
    """N2 (R17): EViT keep mask from padded q, k, v [B, N, H, d]
    (head-averaged CLS logits, CLS + top-(k_keep-2) + one fused token written
    IN PLACE into the first dropped position of q, k and v) -> uint8 keep [B, N]."""
    p = _padded_problem(q, k, v, ENGINE_AUTO, n_hint)
    B, N = q.shape[0], q.shape[1]
    keep = torch.empty(B, N, dtype=torch.uint8, device=q.device) if keep is None else keep
    _require(keep, "keep", torch.uint8, q.device, shape=(B, N))
    _check(lib().ragged_keep_evit(ctypes.byref(p), q.data_ptr(), k.data_ptr(), v.data_ptr(), int(k_keep),
                                  keep.data_ptr(), _stream(stream)), "ragged_keep_evit")
    return keep


def empty_launch(grid: int = 1, block: int = 32, stream=None):
    """Launch-floor probe."""
    _check(lib().ragged_empty_launch(grid, block, _stream(stream)), "ragged_empty_launch")


def validate_cu_seqlens(cu, total: int) -> int:
    """SPEC validate_cu_seqlens, host only: -1 if valid, else the
    first violating index."""
    arr = (ctypes.c_int32 * len(cu))(*[int(x) for x in cu])
    return int(lib().ragged_validate_cu_seqlens(arr, len(cu), int(total)))
