"""Thin ctypes binding of include/ne.h -- argument marshalling only.

Every function keeps the C name; arrays are numpy (host) or torch tensors
(device or pinned host), passed by pointer.  Every step of the training path
runs in libne_b200.so's CUDA kernels; there is no Python or CPU fallback: if
the library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libne_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                      "g.build()'` (nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(LIB_PATH)

NE_OK, NE_EINVAL, NE_ERANGE, NE_ENOMEM, NE_ESTATE, NE_ECUDA, NE_ENCCL, NE_ESCHED = 0, -1, -2, -3, -4, -5, -6, -7
NE_REUSE_SAMPLES = 1
NE_CHECK_BLOCKS = 2
NE_VERTEX, NE_CONTEXT = 0, 1
NE_WB_ATOMIC_DELTA, NE_WB_STORE = 0, 1
NE_UPDATE_SEQUENTIAL, NE_UPDATE_ACCUMULATED, NE_UPDATE_SHARED_BATCH = 0, 1, 2
NE_STAGE_DEVICE, NE_STAGE_HOST = 0, 1
NE_STORE_F32, NE_STORE_BF16 = 0, 1
NE_TRANSPORT_NCCL, NE_TRANSPORT_IPC = 0, 1
NE_STREAM_OWN = (1 << 64) - 1  # ne.h: ((void *)~(uintptr_t)0), the context's own stream


class ne_config(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("negatives", C.c_uint32), ("walk_len", C.c_uint32),
                ("window", C.c_uint32), ("walks_per_node", C.c_uint32), ("episodes", C.c_uint32),
                ("subparts", C.c_uint32), ("deterministic", C.c_uint32), ("conflict_permille", C.c_uint32),
                ("writeback", C.c_uint32), ("p", C.c_float), ("q", C.c_float),
                ("update_rule", C.c_uint32), ("staging", C.c_uint32), ("storage", C.c_uint32),
                ("transport", C.c_uint32), ("seed", C.c_uint64), ("stage_window", C.c_uint32),
                ("groups", C.c_uint32)]


class ne_stats(C.Structure):
    _fields_ = [("samples", C.c_uint64), ("loss_sum", C.c_double), ("ms_walk", C.c_float),
                ("ms_build", C.c_float), ("ms_train", C.c_float), ("ms_comm_wait", C.c_float),
                ("train_launches", C.c_uint32), ("kernel_launches", C.c_uint32), ("ms_pool_wait", C.c_float)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p, C.c_void_p)

_P = C.c_void_p
_sig = {
    "ne_version": (C.c_int, []),
    "ne_create": (C.c_int, [C.POINTER(_P), C.POINTER(ne_config), C.c_int, ALLOC_FN, FREE_FN, _P]),
    "ne_set_stream": (C.c_int, [_P, _P]),
    "ne_join": (C.c_int, [_P]),
    "ne_get_nccl_id": (C.c_int, [_P]),
    "ne_init_dist": (C.c_int, [_P, C.c_int, C.c_int, _P]),
    "ne_load_graph": (C.c_int, [_P, C.c_uint32, C.c_uint64, _P, _P]),
    "ne_random_walk": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, C.c_size_t, C.POINTER(C.c_uint64)]),
    "ne_build_samples": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]),
    "ne_train_samples": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_float, C.POINTER(ne_stats)]),
    "ne_train_epoch": (C.c_int, [_P, C.c_uint32, C.c_float, C.c_uint32, C.POINTER(ne_stats)]),
    "ne_get_embeddings": (C.c_int, [_P, C.c_int, C.c_uint32, C.c_uint32, _P, C.c_size_t]),
    "ne_export_vertex_on_train": (C.c_int, [_P, _P, C.c_size_t]),
    "ne_set_embeddings": (C.c_int, [_P, C.c_int, C.c_uint32, C.c_uint32, _P]),
    "ne_last_error": (C.c_char_p, [_P]),
    "ne_destroy": (None, [_P]),
    "ne_check_pool": (C.c_int, [_P]),
    "ne_export_samples": (C.c_int, [_P, C.c_uint32, _P, C.c_size_t, C.POINTER(C.c_uint64)]),
    "ne_export_negatives": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64, _P]),
    "ne_capture_block": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float, _P, C.c_size_t,
                                   C.POINTER(C.c_uint64)]),
    "ne_ipc_blob_size": (C.c_size_t, []),
    "ne_ipc_export": (C.c_int, [_P, _P, C.c_size_t]),
    "ne_ipc_connect": (C.c_int, [_P, _P, C.c_size_t]),
    "ne_umma_products": (C.c_int, [_P] * 6),
    "ne_umma_raw": (C.c_int, [_P, _P, C.c_uint32, C.c_uint64, C.c_uint64] + [C.c_uint32] * 9 + [_P]),
    "ne_train_samples_local_ring": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32, C.c_float,
                                             C.POINTER(ne_stats)]),
    "ne_plan_vsub": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "ne_partition_bounds": (C.c_int, [C.c_uint64, C.c_uint32, _P]),
    "ne_plan_vsub2": (C.c_int, [C.c_uint32] * 6),
    "ne_ring_peers": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32),
                                C.POINTER(C.c_uint32)]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sig)


class NEError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg or f"NE error {code}")
        self.code = code


def _check(ctx, rc: int) -> None:
    if rc != NE_OK:
        raise NEError(rc, _lib.ne_last_error(ctx).decode())


def _ptr(a, itemsize: int | None = None, what: str = "array") -> int:
    """Address of a C-contiguous numpy array or torch tensor (host or device);
    with `itemsize`, the element size the C side reads (a wrong one would make
    it read past the end of the buffer)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ValueError(f"{what} must be C-contiguous")
        if itemsize is not None and a.itemsize != itemsize:
            raise TypeError(f"{what} has {a.itemsize}-byte elements, the ABI reads {itemsize}-byte ones")
        return a.ctypes.data
    if not a.is_contiguous():  # torch.Tensor
        raise ValueError(f"{what} must be contiguous")
    if itemsize is not None and a.element_size() != itemsize:
        raise TypeError(f"{what} has {a.element_size()}-byte elements, the ABI reads {itemsize}-byte ones")
    return a.data_ptr()


# ---------------------------------------------------------------- ABI, same names
def ne_version() -> int:
    return _lib.ne_version()


def ne_create(cfg: ne_config, device: int, alloc=None, free_fn=None):
    ctx = _P()
    rc = _lib.ne_create(C.byref(ctx), C.byref(cfg), device, alloc or ALLOC_FN(), free_fn or FREE_FN(), None)
    if rc != NE_OK:
        raise NEError(rc, _lib.ne_last_error(None).decode())
    return ctx


def ne_set_stream(ctx, stream: int | None) -> None:
    """stream: a cudaStream_t handle (0 = the legacy default stream, torch's
    default stream) or NE_STREAM_OWN."""
    _check(ctx, _lib.ne_set_stream(ctx, stream))


def ne_join(ctx) -> None:
    _check(ctx, _lib.ne_join(ctx))


def ne_get_nccl_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = _lib.ne_get_nccl_id(buf)
    if rc != NE_OK:
        raise NEError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def ne_init_dist(ctx, rank: int, world: int, nccl_id: bytes | None) -> None:
    buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id else None
    _check(ctx, _lib.ne_init_dist(ctx, rank, world, buf))


def ne_load_graph(ctx, offsets, targets) -> None:
    n = len(offsets) - 1
    nnz = len(targets)
    _check(ctx, _lib.ne_load_graph(ctx, n, nnz, _ptr(offsets, 8, "offsets (u64)"),
                                   _ptr(targets, 4, "targets (u32)") if nnz else None))


def ne_random_walk(ctx, epoch: int, episode: int, host_walks: np.ndarray | None = None) -> int:
    cnt = C.c_uint64()
    cap = host_walks.size if host_walks is not None else 0
    _check(ctx, _lib.ne_random_walk(ctx, epoch, episode, _ptr(host_walks, 4, "host_walks"), cap, C.byref(cnt)))
    return int(cnt.value)


def ne_build_samples(ctx, epoch: int, episode: int) -> int:
    cnt = C.c_uint64()
    _check(ctx, _lib.ne_build_samples(ctx, epoch, episode, C.byref(cnt)))
    return int(cnt.value)


def ne_train_samples(ctx, epoch: int, episode: int, lr: float) -> ne_stats:
    st = ne_stats()
    _check(ctx, _lib.ne_train_samples(ctx, epoch, episode, lr, C.byref(st)))
    return st


def ne_train_epoch(ctx, epoch: int, lr: float, flags: int = 0) -> ne_stats:
    st = ne_stats()
    _check(ctx, _lib.ne_train_epoch(ctx, epoch, lr, flags, C.byref(st)))
    return st


def ne_get_embeddings(ctx, which: int, row_begin: int, row_end: int, out) -> None:
    cap = out.numel() if hasattr(out, "numel") else out.size
    _check(ctx, _lib.ne_get_embeddings(ctx, which, row_begin, row_end, _ptr(out, 4, "out (f32)"), cap))


def ne_export_vertex_on_train(ctx, out) -> None:
    """out: this rank's vertex rows (float32, part rows x d, pinned for the overlap), or None."""
    if out is None:
        _check(ctx, _lib.ne_export_vertex_on_train(ctx, None, 0))
        return
    cap = out.numel() if hasattr(out, "numel") else out.size
    _check(ctx, _lib.ne_export_vertex_on_train(ctx, _ptr(out, 4, "out (f32)"), cap))


def ne_set_embeddings(ctx, which: int, row_begin: int, row_end: int, data) -> None:
    _check(ctx, _lib.ne_set_embeddings(ctx, which, row_begin, row_end, _ptr(data, 4, "data (f32)")))


def ne_last_error(ctx) -> str:
    return _lib.ne_last_error(ctx).decode()


def ne_destroy(ctx) -> None:
    _lib.ne_destroy(ctx)


def ne_check_pool(ctx) -> None:
    _check(ctx, _lib.ne_check_pool(ctx))


def ne_export_samples(ctx, vsub: int, out: np.ndarray | None = None) -> int:
    cnt = C.c_uint64()
    cap = out.size // 2 if out is not None else 0
    _check(ctx, _lib.ne_export_samples(ctx, vsub, _ptr(out, 4, "out (u32 pairs)"), cap, C.byref(cnt)))
    return int(cnt.value)


def ne_export_negatives(ctx, epoch: int, episode: int, vsub: int, pos_begin: int, count: int,
                        out: np.ndarray) -> None:
    _check(ctx, _lib.ne_export_negatives(ctx, epoch, episode, vsub, pos_begin, count, _ptr(out, 4, "out (u32)")))


def ne_capture_block(ctx, epoch: int, episode: int, vsub: int, lr: float, out: np.ndarray | None = None) -> int:
    """Test hook: production-kernel training of one home block, recording
    (src, dst, negatives) per position into out ([count, 2+K] u32)."""
    cnt = C.c_uint64()
    cap = out.size if out is not None else 0
    _check(ctx, _lib.ne_capture_block(ctx, epoch, episode, vsub, lr, _ptr(out, 4, "out (u32)"), cap,
                                      C.byref(cnt)))
    return int(cnt.value)


def ne_ipc_export(ctx) -> bytes:
    n = _lib.ne_ipc_blob_size()
    buf = (C.c_uint8 * n)()
    _check(ctx, _lib.ne_ipc_export(ctx, buf, n))
    return bytes(buf)


def ne_ipc_connect(ctx, blobs: list[bytes]) -> None:
    n = _lib.ne_ipc_blob_size()
    assert all(len(b) == n for b in blobs)
    buf = (C.c_uint8 * (n * len(blobs))).from_buffer_copy(b"".join(blobs))
    _check(ctx, _lib.ne_ipc_connect(ctx, buf, n))


def ne_umma_products(V, N, G):
    """Test hook: the tcgen05 products of the batch kernel; returns (S, dV, dNt)."""
    V, N, G = (np.ascontiguousarray(x, np.float32) for x in (V, N, G))
    assert V.shape == (128, 128) and N.shape == (32, 128) and G.shape == (128, 32)
    S, dV, dNt = np.zeros((128, 32), np.float32), np.zeros((128, 128), np.float32), np.zeros((128, 32), np.float32)
    rc = _lib.ne_umma_products(_ptr(V), _ptr(N), _ptr(G), _ptr(S), _ptr(dV), _ptr(dNt))
    if rc != NE_OK:
        raise NEError(rc, "ne_umma_products failed")
    return S, dV, dNt


def ne_umma_raw(a_img: bytes, b_img: bytes, a_hi: int, b_hi: int, a_lbo: int, a_sbo: int, b_lbo: int, b_sbo: int,
                a_step: int, b_step: int, ksteps: int, idesc: int, N: int) -> np.ndarray:
    """Diagnostics hook: one tcgen05 tf32 product from raw smem images."""
    assert len(a_img) == len(b_img) and len(a_img) % 16 == 0
    D = np.zeros((128, N), np.float32)
    ab, bb = (C.c_char * len(a_img)).from_buffer_copy(a_img), (C.c_char * len(b_img)).from_buffer_copy(b_img)
    rc = _lib.ne_umma_raw(C.cast(ab, _P), C.cast(bb, _P), len(a_img), a_hi, b_hi, a_lbo, a_sbo, b_lbo, b_sbo, a_step,
                          b_step, ksteps, idesc, N, _ptr(D))
    if rc != NE_OK:
        raise NEError(rc, "ne_umma_raw failed")
    return D


def ne_train_samples_local_ring(ctxs, epoch: int, episode: int, lr: float) -> ne_stats:
    arr = (_P * len(ctxs))(*[c.value for c in ctxs])
    st = ne_stats()
    _check(ctxs[0], _lib.ne_train_samples_local_ring(arr, len(ctxs), epoch, episode, lr, C.byref(st)))
    return st


def ne_plan_vsub(world: int, subparts: int, r: int, t: int, g: int) -> int:
    return _lib.ne_plan_vsub(world, subparts, r, t, g)


def ne_plan_vsub2(world: int, groups: int, subparts: int, rho: int, t: int, g: int) -> int:
    return _lib.ne_plan_vsub2(world, groups, subparts, rho, t, g)


def ne_ring_peers(world: int, groups: int, rho: int, g: int) -> tuple[int, int]:
    d, s_ = C.c_uint32(), C.c_uint32()
    if _lib.ne_ring_peers(world, groups, rho, g, C.byref(d), C.byref(s_)) != NE_OK:
        raise NEError(NE_EINVAL, "bad ring arguments")
    return int(d.value), int(s_.value)


def ne_partition_bounds(n: int, parts: int) -> np.ndarray:
    b = np.zeros(parts + 1, np.uint64)
    rc = _lib.ne_partition_bounds(n, parts, b.ctypes.data)
    if rc != NE_OK:
        raise NEError(rc, "bad partition arguments")
    return b


# ---------------------------------------------------------------- torch allocator
def torch_allocator():
    """(alloc, free) callbacks routing device memory through PyTorch's caching
    allocator (keep the returned objects alive as long as the context)."""
    import torch

    def _alloc(nbytes, device, stream, user):
        try:
            return torch.cuda.caching_allocator_alloc(nbytes, device, stream or 0)
        except Exception:  # out of memory -> NULL -> NE_ENOMEM
            return None

    def _free(ptr, nbytes, device, stream, user):
        torch.cuda.caching_allocator_delete(ptr)

    return ALLOC_FN(_alloc), FREE_FN(_free)
