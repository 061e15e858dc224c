"""C-ABI checks that need no GPU: the library loads, exports every entry point
include/ragged.h declares, and rejects every host-checkable bad argument with
the documented status BEFORE touching CUDA."""
import ctypes
import json
import os
import re
import subprocess

import pytest
import torch

from conftest import GOLDEN, ROOT

rb = pytest.importorskip("paper_2604_15408_b200")


def _declared():
    # ragged_debug.h declares the timeline-build-only symbols (libragged_tl.so).
    src = "".join(open(os.path.join(ROOT, "include", h)).read()
                  for h in ("ragged.h", "ragged_dist.h", "ragged_block.h"))
    return sorted(set(re.findall(r"^\s*RAGGED_API\s+(?:ragged_status|void|int32_t|int64_t|const char\*)\s+(ragged_\w+)\(",
                                 src, re.M)))


def test_header_and_library_exports_agree():
    names = _declared()
    assert len(names) >= 12
    for n in names:
        assert hasattr(rb.lib(), n), n
    assert set(names) == set(rb.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", rb.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\b(ragged_\w+)\b", out))
    assert set(names) <= exported
    assert not [s for s in exported if s not in names], "undeclared ragged_* symbols exported"


def test_library_targets_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", rb.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_100a" in rb.build_info()


def test_status_strings():
    for code, name in [(0, "RAGGED_OK"), (1, "RAGGED_EINVAL"), (2, "RAGGED_ENOTSUP"), (3, "RAGGED_EALIGN"),
                       (4, "RAGGED_ECUDA")]:
        assert rb.status_str(code) == name
    assert rb.status_str(99) == "RAGGED_UNKNOWN"


FAKE = 0x10000  # 16-byte aligned, never dereferenced (validation fails or B == 0 first)


def _call_fused(p, keep=FAKE, q=FAKE, k=FAKE, v=FAKE, o=FAKE):
    return rb.lib().ragged_pack_attend_unpack(ctypes.byref(p), keep, q, k, v, o, None, None)


@pytest.mark.parametrize("field,value,status", [
    ("B", -1, rb.EINVAL), ("N", 0, rb.EINVAL), ("H", 0, rb.EINVAL), ("N", 257, rb.ENOTSUP),
    ("d", 128, rb.ENOTSUP), ("dtype", 7, rb.ENOTSUP), ("engine", 9, rb.ENOTSUP),
    ("ld", 100, rb.EINVAL), ("ld", 772, rb.EALIGN), ("n_hint", -1, rb.EINVAL),
])
def test_problem_validation(field, value, status):
    p = rb.problem(4, 197, 12)
    setattr(p, field, value)
    assert _call_fused(p) == status
    assert rb.last_error() != ""


def test_pointer_validation():
    p = rb.problem(4, 197, 12)
    assert _call_fused(p, q=0) == rb.EINVAL
    assert _call_fused(p, keep=0) == rb.EINVAL
    assert _call_fused(p, o=FAKE + 2) == rb.EALIGN
    assert rb.lib().ragged_attn(ctypes.byref(p), FAKE, FAKE, FAKE + 8, FAKE, FAKE, None) == rb.EALIGN
    assert rb.lib().ragged_unpack(ctypes.byref(p), FAKE, None, FAKE, None) == rb.EINVAL
    assert rb.lib().ragged_scan(ctypes.byref(p), FAKE, None, FAKE, FAKE, None) == rb.EINVAL
    assert rb.lib().ragged_pack(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, FAKE,
                                FAKE, FAKE, FAKE + 4, None) == rb.EALIGN
    assert rb.lib().ragged_scan(None, FAKE, FAKE, FAKE, FAKE, None) == rb.EINVAL
    h = ctypes.c_void_p()
    assert rb.lib().ragged_graph_create(None, FAKE, FAKE, FAKE, FAKE, FAKE, None, ctypes.byref(h)) == rb.EINVAL
    assert rb.lib().ragged_graph_create(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE, FAKE, None, None) == rb.EINVAL
    assert rb.lib().ragged_graph_launch(None, None) == rb.EINVAL
    rb.lib().ragged_graph_destroy(None)
    assert rb.lib().ragged_empty_launch(0, 32, None) == rb.EINVAL


def test_host_entry_validation():
    """ragged_pack_attend_unpack_host: host-checkable errors before any CUDA call."""
    f = rb.lib().ragged_pack_attend_unpack_host
    p = rb.problem(4, 197, 12)
    assert f(ctypes.byref(p), FAKE, 0, FAKE, FAKE, FAKE, None, None) == rb.EINVAL
    assert f(ctypes.byref(p), 0, FAKE, FAKE, FAKE, FAKE, None, None) == rb.EINVAL
    assert f(ctypes.byref(p), FAKE, FAKE, FAKE + 8, FAKE, FAKE, None, None) == rb.EALIGN
    assert f(None, FAKE, FAKE, FAKE, FAKE, FAKE, None, None) == rb.EINVAL
    p.d = 32
    assert f(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE, FAKE, None, None) == rb.ENOTSUP
    assert f(ctypes.byref(rb.problem(0, 197, 12)), None, None, None, None, None, None, None) == rb.OK
    with pytest.raises(ValueError):   # the binding takes pinned CPU tensors only
        t = torch.zeros(1, 197, 12, 64, dtype=torch.bfloat16)
        rb.pack_attend_unpack_host(t, t, t, torch.ones(1, 197, dtype=torch.uint8), t)


def _gather_call(p, g, fused=True):
    if fused:
        return rb.lib().ragged_pack_attend_unpack_gather(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE, None,
                                                         ctypes.byref(g) if g is not None else None, None)
    return rb.lib().ragged_attn_gather(ctypes.byref(p), FAKE, FAKE, FAKE, FAKE,
                                       ctypes.byref(g) if g is not None else None, None)


def test_gather_validation():
    """ragged_dist.h: every host-checkable gather error, before any CUDA call
    (B = 0 reaches the no-op return only after the descriptor is valid)."""
    p = rb.problem(0, 197, 12)
    ok = rb.gather_desc(2, 1, out=[FAKE, FAKE])
    assert _gather_call(p, ok) == rb.OK
    assert _gather_call(p, ok, fused=False) == rb.OK
    assert _gather_call(p, None) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(0, 0)) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(9, 0)) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(2, 2, out=[FAKE, FAKE])) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(2, -1, out=[FAKE, FAKE])) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(2, 0)) == rb.EINVAL                       # no destination
    assert _gather_call(p, rb.gather_desc(2, 0, out=[FAKE, FAKE + 8])) == rb.EALIGN
    assert _gather_call(p, rb.gather_desc(2, 0, cls=[FAKE + 4, None])) == rb.EALIGN
    assert _gather_call(p, rb.gather_desc(2, 0, cls=[FAKE, FAKE]), fused=False) == rb.EINVAL
    # signals must cover every rank and come with state
    assert _gather_call(p, rb.gather_desc(2, 0, out=[FAKE, FAKE], signal=[FAKE, None], state=FAKE)) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(2, 0, out=[FAKE, FAKE], signal=[FAKE, FAKE])) == rb.EINVAL
    assert _gather_call(p, rb.gather_desc(2, 0, out=[FAKE, FAKE], signal=[FAKE, FAKE], state=FAKE)) == rb.OK
    p2 = rb.problem(0, 197, 12, engine=rb.ENGINE_TCGEN05)
    assert _gather_call(p2, ok) == rb.ENOTSUP
    with pytest.raises(ValueError):
        rb.gather_desc(2, 0, out=[FAKE])


def test_empty_batch_is_noop_without_cuda():
    """B == 0 returns OK and launches nothing (no CUDA device here)."""
    p = rb.problem(0, 197, 12)
    assert _call_fused(p, q=0, k=0, v=0, o=0, keep=0) == rb.OK
    assert rb.lib().ragged_scan(ctypes.byref(p), None, None, None, None, None) == rb.OK
    assert rb.lib().ragged_attn(ctypes.byref(p), None, None, None, None, None, None) == rb.OK


def test_validate_cu_seqlens_spec_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_scan_examples.json")))
    for c in g["valid_cu"]:
        assert rb.validate_cu_seqlens(c["cu"], c["T"]) == -1
    assert rb.validate_cu_seqlens([0, 5, 3], 3) == 2          # non-monotone at index 2
    assert rb.validate_cu_seqlens([1, 5], 5) == 0
    assert rb.validate_cu_seqlens([0, 5, 6], 7) == 2


def test_python_binding_rejects_bad_layouts():
    import torch
    q = torch.zeros(2, 5, 3, 64, dtype=torch.float32)
    with pytest.raises(ValueError):
        rb.pack_attend_unpack(q, q, q, torch.ones(2, 5, dtype=torch.uint8))
    qb = torch.zeros(2, 5, 3, 64, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        rb.pack_attend_unpack(qb, qb.transpose(0, 1).contiguous().transpose(0, 1), qb,
                              torch.ones(2, 5, dtype=torch.uint8))
    with pytest.raises(ValueError):
        rb.pack_attend_unpack(qb, qb, qb, torch.ones(2, 5, dtype=torch.int32))


def test_product_package_does_not_import_oracle():
    """The product path never routes through the oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2604_15408_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle/", ""), f


def test_general_attn_validation():
    """ragged_attn's widened shapes (NEXT row N4) pass validation; the fused /
    pack / unpack paths keep the DeiT caps."""
    L = rb.lib()
    for d in (32, 80, 128):
        p = rb.problem(0, 1000, 4, d=d)
        assert L.ragged_attn(ctypes.byref(p), None, None, None, None, None, None) == rb.OK
    assert L.ragged_attn(ctypes.byref(rb.problem(0, 197, 4, d=96)), None, None, None, None, None, None) == rb.ENOTSUP
    assert L.ragged_attn(ctypes.byref(rb.problem(0, (1 << 20) + 1, 1)), None, None, None, None, None,
                         None) == rb.ENOTSUP
    assert _call_fused(rb.problem(0, 300, 4)) == rb.ENOTSUP
    assert _call_fused(rb.problem(0, 197, 4, d=128)) == rb.ENOTSUP


def test_block_validation():
    """ragged_block.h host-checkable errors (no CUDA call)."""
    L = rb.lib()
    assert L.ragged_layer_norm(0, 4, 12, FAKE, 12, FAKE, FAKE, 1e-6, FAKE, 12, None, None) == rb.EINVAL  # D % 8
    assert L.ragged_layer_norm(0, 4, 2048, FAKE, 2048, FAKE, FAKE, 1e-6, FAKE, 2048, None, None) == rb.EINVAL
    assert L.ragged_layer_norm(0, 4, 64, FAKE, 60, FAKE, FAKE, 1e-6, FAKE, 64, None, None) == rb.EINVAL
    assert L.ragged_layer_norm(0, 4, 64, FAKE + 2, 64, FAKE, FAKE, 1e-6, FAKE, 64, None, None) == rb.EALIGN
    assert L.ragged_layer_norm(5, 4, 64, FAKE, 64, FAKE, FAKE, 1e-6, FAKE, 64, None, None) == rb.ENOTSUP
    assert L.ragged_layer_norm(0, 0, 64, None, 64, None, None, 1e-6, None, 64, None, None) == rb.OK
    lin = lambda *a: L.ragged_linear(*a, None, None)  # noqa: E731
    assert lin(0, 4, 100, 64, FAKE, 64, FAKE, None, 0, None, 0, FAKE, 100) == rb.ENOTSUP       # N % 64
    assert lin(0, 4, 64, 96, FAKE, 96, FAKE, None, 0, None, 0, FAKE, 64) == rb.ENOTSUP         # K % 64
    assert lin(0, 4, 64, 64, FAKE, 64, FAKE, None, 7, None, 0, FAKE, 64) == rb.EINVAL          # epilogue
    assert lin(0, 4, 64, 64, FAKE, 64, FAKE, None, 2, None, 64, FAKE, 64) == rb.EINVAL         # residual NULL
    assert lin(0, 4, 64, 64, FAKE, 64, FAKE, FAKE + 4, 0, None, 0, FAKE, 64) == rb.EALIGN      # bias
    assert lin(0, 4, 64, 64, FAKE, 60, FAKE, None, 0, None, 0, FAKE, 64) == rb.EINVAL          # lda < K
    assert lin(0, 0, 64, 64, None, 64, None, None, 0, None, 0, None, 64) == rb.OK
    p = rb.problem(4, 197, 12)
    assert L.ragged_vit_block_workspace(ctypes.byref(p), 3072) == 4 * 197 * (5 * 768 + 3072) * 2
    assert L.ragged_vit_block_workspace(ctypes.byref(rb.problem(4, 197, 12, d=32)), 3072) == -1
    w = rb.VitWeights()
    w.mlp = 3072
    assert L.ragged_vit_block(ctypes.byref(p), FAKE, FAKE, ctypes.byref(w), FAKE, 10, None) == rb.EINVAL  # ws
    big = 1 << 40
    assert L.ragged_vit_block(ctypes.byref(p), FAKE, FAKE, ctypes.byref(w), FAKE, big, None) == rb.EINVAL  # NULL w
    w.mlp = 100
    assert L.ragged_vit_block(ctypes.byref(p), FAKE, FAKE, ctypes.byref(w), FAKE, big, None) == rb.ENOTSUP
    assert L.ragged_vit_block(None, FAKE, FAKE, ctypes.byref(w), FAKE, big, None) == rb.EINVAL


def test_python_binding_checks_caller_buffers():
    """the ABI cannot see buffer sizes, so the binding checks every
    caller buffer (shape, dtype, device, size) before a pointer crosses it.
    CPU tensors suffice: every check fires before any library call."""
    import torch
    B, N, H, d = 2, 5, 3, 64
    q = torch.zeros(B, N, H, d, dtype=torch.bfloat16)
    keep = torch.ones(B, N, dtype=torch.uint8)
    bad = [
        lambda: rb.pack_attend_unpack(q, q, q, torch.ones(B, N + 1, dtype=torch.uint8)),   # mask shape
        lambda: rb.pack_attend_unpack(q, q, q, keep, o=torch.zeros(B, N, H, d - 8, dtype=torch.bfloat16)),
        lambda: rb.pack_attend_unpack(q, q, q, keep, o=torch.zeros(B, N, H, d, dtype=torch.float16)),
        lambda: rb.pack_attend_unpack(q, q, q, keep, cu=torch.zeros(B + 1, dtype=torch.int64)),
        lambda: rb.pack_attend_unpack(q, q, q, keep, cu=torch.zeros(B, dtype=torch.int32)),
        lambda: rb.scan(keep, cu=torch.zeros(B, dtype=torch.int32)),
        lambda: rb.scan(keep, dst=torch.zeros(B * N - 1, dtype=torch.int32)),
        lambda: rb.pack(q, q, q, keep, out=(torch.zeros(B * N - 1, H, d, dtype=torch.bfloat16),) * 3
                        + (torch.zeros(B + 1, dtype=torch.int32), torch.zeros(B * N, dtype=torch.int32),
                           torch.zeros(B * N, dtype=torch.int32))),
        lambda: rb.attn(*(torch.zeros(B * N - 1, H, d, dtype=torch.bfloat16),) * 3, torch.zeros(B + 1, dtype=torch.int32), N),
        lambda: rb.attn(*(torch.zeros(B * N, H, d, dtype=torch.bfloat16),) * 3, torch.zeros(B + 1, dtype=torch.int64), N),
        lambda: rb.attn(*(torch.zeros(B * N, H, d, dtype=torch.bfloat16),) * 3, torch.zeros(B + 1, dtype=torch.int32), N,
                        op=torch.zeros(B * N - 1, H, d, dtype=torch.bfloat16)),
        lambda: rb.unpack(torch.zeros(B * N, H, d, dtype=torch.bfloat16), torch.zeros(B * N - 1, dtype=torch.int32), B, N),
        lambda: rb.unpack(torch.zeros(B * N, H, d, dtype=torch.bfloat16), torch.zeros(B * N, dtype=torch.int32), B, N,
                          o=torch.zeros(B, N, H, d // 2, dtype=torch.bfloat16)),
        lambda: rb.keep_topk_l2(torch.zeros(B, N, 128, dtype=torch.bfloat16), 3, keep=torch.zeros(B, N - 1, dtype=torch.uint8)),
    ]
    for i, f in enumerate(bad):
        with pytest.raises(ValueError):
            f()


def test_dist_nccl_entry_validation():
    """NCCL entry points: NULL / range checks return synchronously; NCCL itself
    is loaded at run time (available or RAGGED_ENOTSUP, never a crash)."""
    import ctypes
    lib = rb.lib()
    assert lib.ragged_dist_nccl_available() in (rb.OK, rb.ENOTSUP)
    assert lib.ragged_dist_nccl_unique_id(None) == rb.EINVAL
    h = ctypes.c_void_p()
    uid = (ctypes.c_uint8 * 128)()
    assert lib.ragged_dist_nccl_init(None, 1, 0, ctypes.byref(h)) == rb.EINVAL
    assert lib.ragged_dist_nccl_init(uid, 2, 2, ctypes.byref(h)) == rb.EINVAL
    assert lib.ragged_dist_nccl_init_all(0, None, None) == rb.EINVAL
    p = rb.problem(2, 197, 12)
    assert lib.ragged_dist_pack_attend_unpack_allgather(ctypes.byref(p), None, None, None, None, None, None, None,
                                                        None, None) == rb.EINVAL
    lib.ragged_dist_nccl_destroy(None)


def test_round2_entry_validation():
    """Round-2 entry points (N2 EViT / fused prune, N1 pack_rows / cls_rows, the
    WS engine): host-checkable errors return synchronously, before any CUDA
    call (FAKE pointers are never dereferenced)."""
    lib = rb.lib()
    p = rb.problem(4, 197, 12)
    # ragged_keep_evit: k < 1, NULL q, H too large for its row buffers at N = 256
    assert lib.ragged_keep_evit(ctypes.byref(p), FAKE, FAKE, FAKE, 0, FAKE, None) == rb.EINVAL
    assert lib.ragged_keep_evit(ctypes.byref(p), None, FAKE, FAKE, 5, FAKE, None) == rb.EINVAL
    big = rb.problem(4, 256, 40)
    assert lib.ragged_keep_evit(ctypes.byref(big), FAKE, FAKE, FAKE, 5, FAKE, None) == rb.ENOTSUP
    assert lib.ragged_keep_evit(ctypes.byref(rb.problem(0, 197, 12)), None, None, None, 5, None, None) == rb.OK
    # ragged_keep_topk_l2: k < 1
    assert lib.ragged_keep_topk_l2(ctypes.byref(p), FAKE, 0, FAKE, None) == rb.EINVAL
    # ragged_prune_l2_pack_attend_unpack: k < 1, H > 16, ldx < H*d, ldx alignment, the WS engine
    f = lib.ragged_prune_l2_pack_attend_unpack
    assert f(ctypes.byref(p), FAKE, 768, 0, FAKE, FAKE, FAKE, FAKE, None, None, None) == rb.EINVAL
    assert f(ctypes.byref(rb.problem(4, 197, 17)), FAKE, 17 * 64, 5, FAKE, FAKE, FAKE, FAKE, None, None,
             None) == rb.ENOTSUP
    assert f(ctypes.byref(p), FAKE, 512, 5, FAKE, FAKE, FAKE, FAKE, None, None, None) == rb.EINVAL
    assert f(ctypes.byref(p), FAKE, 772, 5, FAKE, FAKE, FAKE, FAKE, None, None, None) == rb.EALIGN
    ws = rb.problem(4, 197, 12, engine=rb.ENGINE_TCGEN05_WS)
    assert f(ctypes.byref(ws), FAKE, 768, 5, FAKE, FAKE, FAKE, FAKE, None, None, None) == rb.ENOTSUP
    # the WS engine's fused path: head_dim 64; a cu_seqlens output only for B*N <= 65536
    big_ws = rb.problem(400, 197, 12, engine=rb.ENGINE_TCGEN05_WS)
    assert lib.ragged_pack_attend_unpack(ctypes.byref(big_ws), FAKE, FAKE, FAKE, FAKE, FAKE, FAKE, None) == rb.ENOTSUP
    ws80f = rb.problem(4, 197, 12, d=80, engine=rb.ENGINE_TCGEN05_WS)
    assert lib.ragged_pack_attend_unpack(ctypes.byref(ws80f), FAKE, FAKE, FAKE, FAKE, FAKE, None, None) in (
        rb.ENOTSUP,)
    ws80 = rb.problem(4, 300, 12, d=80, engine=rb.ENGINE_TCGEN05_WS)
    assert lib.ragged_attn(ctypes.byref(ws80), FAKE, FAKE, FAKE, FAKE, FAKE, None) == rb.ENOTSUP
    # N1 pieces: NULL pointers
    assert lib.ragged_pack_rows(ctypes.byref(p), FAKE, None, FAKE, FAKE, FAKE, FAKE, None) == rb.EINVAL
    assert lib.ragged_cls_rows(ctypes.byref(p), FAKE, FAKE, None, None) == rb.EINVAL
