"""Python binding of libheatfem.so -- the B200 hot path of arXiv 1905.07622.

Thin ctypes marshalling over the C ABI of ``include/heatfem.h`` with the SAME function
names.  Every computation runs in the library's sm_100a kernels; this module only checks
dtypes/sizes and passes pointers.  There is no CPU fallback: importing fails loudly when
the shared library is missing (build it with ``python -m paper_1905_07622_b200._build``).

Arrays may be torch tensors (CUDA or CPU) or numpy arrays, float64 and contiguous.  CUDA
tensors are passed by device pointer on the current torch stream; host arrays are staged
by the library itself.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.environ.get("HF_LIB_VARIANT") or os.path.join(_HERE, "libheatfem.so")   # variant: A/B experiments

if not os.path.exists(_LIB_PATH):
    raise ImportError(f"libheatfem.so not built ({_LIB_PATH}); run python -m paper_1905_07622_b200._build")

HF_OK, HF_E_ARG, HF_E_INDEX, HF_E_NOCONV, HF_E_BREAKDOWN = 0, -1, -2, -3, -4
HF_E_PARTITION, HF_E_CUDA, HF_E_NCCL, HF_E_OOM, HF_E_STATE = -5, -6, -7, -8, -9
FACE_XM, FACE_XP, FACE_YM, FACE_YP, FACE_ZM, FACE_ZP = range(6)


class HfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"heatfem status {status}: {msg}")
        self.status = status


class hf_grid(C.Structure):
    _fields_ = [("ne", C.c_int64 * 3), ("h", C.c_double * 3), ("origin", C.c_double * 3)]


class hf_cg_opts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iter", C.c_int32), ("replace_every", C.c_int32)]


class hf_cg_info(C.Structure):
    _fields_ = [("iters", C.c_int32), ("status", C.c_int32), ("relres", C.c_double), ("delta", C.c_double)]


class hf_sim_stats(C.Structure):
    _fields_ = [("steps_done", C.c_int32), ("total_iters", C.c_int32), ("max_iters_step", C.c_int32),
                ("first_failed_step", C.c_int32), ("ms_total", C.c_double), ("ms_steps", C.c_double)]


_lib = C.CDLL(_LIB_PATH)
_vp, _dp, _i32, _i64, _d = C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_double
_P = C.POINTER

_SIGS = {
    "hf_version": (C.c_char_p, []),
    "hf_last_error": (C.c_char_p, []),
    "hf_create": (_i32, [_P(hf_grid), C.c_int, _vp, _P(_vp)]),
    "hf_destroy": (None, [_vp]),
    "hf_set_coefficients": (_i32, [_vp, _dp, _dp]),
    "hf_set_dirichlet_faces": (_i32, [_vp, C.c_uint32, _P(C.c_double * 6)]),
    "hf_face_load": (_i32, [_vp, C.c_int, _d, _P(C.c_double * 4), _dp]),
    "hf_apply": (_i32, [_vp, _d, _d, _dp, _dp]),
    "hf_apply_axpby": (_i32, [_vp, _d, _d, _d, _dp, _dp, _dp]),
    "hf_diag": (_i32, [_vp, _d, _d, _dp]),
    "hf_cg": (_i32, [_vp, _d, _d, _dp, _dp, _P(hf_cg_opts), _P(hf_cg_info)]),
    "hf_simulate": (_i32, [_vp, _d, _d, _i32, _dp, _dp, _i64, _dp, _P(hf_cg_opts), _P(hf_sim_stats)]),
    "hf_simulate_resume": (_i32, [_vp, _d, _d, _i32, _dp, _dp, _dp, _i64, _P(hf_cg_opts), _P(hf_sim_stats)]),
    "hf_simulate_batched": (_i32, [_vp, _i32, _dp, _dp, _d, _d, _i32, _dp, _dp, _i64, _dp, _P(hf_cg_opts),
                                   _P(hf_sim_stats)]),
    "hf_slab_plan": (_i32, [_i64, _i32, _i32, _P(_i64), _P(_i64)]),
    "hf_nccl_unique_id": (_i32, [C.c_char_p]),
    "hf_create_slab": (_i32, [_P(hf_grid), _i32, _i32, _vp, _i32, C.c_int, _vp, _P(_vp)]),
    "hf_local_group_create": (_i32, [_i32, _P(_vp)]),
    "hf_local_group_destroy": (None, [_vp]),
    "hf_peer_export": (_i32, [_vp, C.c_char_p]),
    "hf_peer_connect": (_i32, [_vp, C.c_char_p]),
    "hf_slab_range": (_i32, [_vp, _P(_i64), _P(_i64), _P(_i64), _P(_i64)]),
    "hf_get_launch_count": (_i32, [_vp, _P(_i64)]),
    "hf_profile": (_i32, [_vp, _i32]),
    "hf_profile_read": (_i32, [_vp, _P(C.c_double * 5), _P(C.c_int64 * 5)]),
    "hf_set_driver": (_i32, [_vp, _i32]),
    "hf_set_resident": (_i32, [_vp, _i32]),
    "hf_set_cg_variant": (_i32, [_vp, _i32]),
    "hf_set_tuning": (_i32, [_vp, C.c_char_p, C.c_int64]),
    "hf_time_kernel_a_graph": (_i32, [_vp, _i32, _P(C.c_double)]),
    "hf_get_tuning": (_i32, [_vp, C.c_char_p, _P(C.c_int64)]),
    "hf_cg_variant": (_i32, [_vp, _P(C.c_int32)]),
    "hf_set_mixed": (_i32, [_vp, _i32, _d]),
    "hf_mixed_iters": (_i32, [_vp, _P(C.c_int64)]),
    "hf_resident_plan": (_i32, [_vp, _P(C.c_int32)]),
    "hf_resident_profile": (_i32, [_vp, _i32, _P(C.c_double)]),
    "hf_flush_l2": (_i32, [_vp]),
    "hf_set_step_flush": (_i32, [_vp, _i32]),
    "hf_set_element": (_i32, [_vp, _i32]),
    "hf_set_precision": (_i32, [_vp, _i32]),
    "hf_set_vertex_coefficients": (_i32, [_vp, _vp, _vp]),
    "hf_time_kernel_a": (_i32, [_vp, _i32, C.POINTER(C.c_double)]),
    "hf_apply_impl": (_i32, [_vp, _i32, _d, _d, _d, _dp, _dp, _dp]),
    "hf_ablation_prepare": (_i32, [_vp, _d, _d]),
    "hf_set_material_ids": (_i32, [_vp, _vp, _i32, _P(C.c_double), _P(C.c_double)]),
}
for _name, (_res, _args) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

ABI_FUNCTIONS = tuple(_SIGS)


def _check(st: int):
    if st != HF_OK:
        raise HfError(st, _lib.hf_last_error().decode())


def _ptr(a, n: Optional[int] = None, name: str = "array", allow_none: bool = False):
    """Pointer of a float64 contiguous torch tensor / numpy array (size check only)."""
    if a is None:
        if allow_none:
            return None
        raise HfError(HF_E_ARG, f"{name} is None")
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise HfError(HF_E_ARG, f"{name}: need a contiguous float64 tensor")
            if n is not None and a.numel() != n:
                raise HfError(HF_E_ARG, f"{name}: {a.numel()} entries, expected {n}")
            return a.data_ptr()
    except ImportError:
        pass
    import numpy as np
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous:
            raise HfError(HF_E_ARG, f"{name}: need a C-contiguous float64 array")
        if n is not None and a.size != n:
            raise HfError(HF_E_ARG, f"{name}: {a.size} entries, expected {n}")
        return a.ctypes.data
    raise HfError(HF_E_ARG, f"{name}: unsupported type {type(a)}")


def _cptr(ctx, a, n: Optional[int] = None, name: str = "array", allow_none: bool = False):
    """_ptr for an array passed to context `ctx`: a CUDA tensor must live on the context's device."""
    try:
        import torch
        if isinstance(a, torch.Tensor) and a.is_cuda and a.device.index != ctx.device:
            raise HfError(HF_E_ARG, f"{name}: tensor on {a.device}, context on cuda:{ctx.device}")
    except ImportError:
        pass
    return _ptr(a, n, name, allow_none)


CUDA_STREAM_LEGACY = 1   # cudaStreamLegacy: torch's default stream reports handle 0


def _stream(stream, device: int):
    """The torch stream the context should enqueue on (its default stream -> cudaStreamLegacy,
    so torch events and synchronisation see the library's work)."""
    if stream is not None:
        return stream
    try:
        import torch
        if torch.cuda.is_available():
            h = torch.cuda.current_stream(device).cuda_stream
            return h if h else CUDA_STREAM_LEGACY
    except ImportError:
        pass
    return None


def _opts(rtol, max_iter, replace_every):
    return hf_cg_opts(rtol, max_iter, replace_every)


def make_grid(grid) -> hf_grid:
    """hf_grid from an object with ne/h/origin attributes, or a (ne, h[, origin]) tuple."""
    if isinstance(grid, hf_grid):
        return grid
    if hasattr(grid, "ne"):
        ne, h, origin = grid.ne, grid.h, getattr(grid, "origin", (0.0, 0.0, 0.0))
    else:
        ne, h = grid[0], grid[1]
        origin = grid[2] if len(grid) > 2 else (0.0, 0.0, 0.0)
    return hf_grid((C.c_int64 * 3)(*ne), (C.c_double * 3)(*h), (C.c_double * 3)(*origin))


class Context:
    """An hf_ctx* plus the sizes the binding checks against."""

    def __init__(self, ptr, grid: hf_grid, device: int, local_planes: int):
        self.ptr = C.c_void_p(ptr)
        self.grid = grid
        self.device = device
        self.ne = tuple(grid.ne)
        self.n_elems = self.ne[0] * self.ne[1] * self.ne[2]
        self.n_plane = (self.ne[0] + 1) * (self.ne[1] + 1)
        self.n_nodes = self.n_plane * local_planes   # local (slab) node count
        self.n_nodes_global = self.n_plane * (self.ne[2] + 1)

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value and _lib is not None:   # (interpreter shutdown)
            _lib.hf_destroy(self.ptr)
            self.ptr = C.c_void_p(None)


# ---- C ABI, same names ---------------------------------------------------------------------

def hf_version() -> str:
    return _lib.hf_version().decode()


def hf_last_error() -> str:
    return _lib.hf_last_error().decode()


def hf_create(grid, device: int = 0, stream=None) -> Context:
    g = make_grid(grid)
    out = C.c_void_p()
    _check(_lib.hf_create(C.byref(g), device, _stream(stream, device), C.byref(out)))
    return Context(out.value, g, device, g.ne[2] + 1)


def hf_destroy(ctx: Context):
    if ctx.ptr.value:
        _lib.hf_destroy(ctx.ptr)
        ctx.ptr = C.c_void_p(None)


def hf_set_coefficients(ctx: Context, k, c):
    _check(_lib.hf_set_coefficients(ctx.ptr, _cptr(ctx, k, ctx.n_elems, "k"), _cptr(ctx, c, ctx.n_elems, "c")))


def hf_set_vertex_coefficients(ctx: Context, k_node, c_node):
    """Per-node materials of the global grid, averaged over each element's vertices."""
    n = ctx.n_nodes_global
    _check(_lib.hf_set_vertex_coefficients(ctx.ptr, _cptr(ctx, k_node, n, "k_node"), _cptr(ctx, c_node, n, "c_node")))


def hf_set_dirichlet_faces(ctx: Context, face_bits: int, values: Optional[Sequence[float]] = None):
    v = (C.c_double * 6)(*(values if values is not None else (0.0,) * 6))
    _check(_lib.hf_set_dirichlet_faces(ctx.ptr, face_bits, C.byref(v)))


def hf_face_load(ctx: Context, face: int, f_const: float, beam, F):
    b = None if beam is None else C.byref((C.c_double * 4)(*beam))
    _check(_lib.hf_face_load(ctx.ptr, face, f_const, b, _cptr(ctx, F, ctx.n_nodes, "F")))


def hf_apply(ctx: Context, aK: float, aM: float, u, y):
    _check(_lib.hf_apply(ctx.ptr, aK, aM, _cptr(ctx, u, ctx.n_nodes, "u"), _cptr(ctx, y, ctx.n_nodes, "y")))


def hf_apply_axpby(ctx: Context, aK: float, aM: float, c: float, u, b, y):
    _check(_lib.hf_apply_axpby(ctx.ptr, aK, aM, c, _cptr(ctx, u, ctx.n_nodes, "u"),
                               _cptr(ctx, b, ctx.n_nodes, "b", allow_none=True), _cptr(ctx, y, ctx.n_nodes, "y")))


def hf_set_material_ids(ctx: Context, ids, k_mat: Sequence[float], c_mat: Sequence[float]):
    """Materials by id: k_e = k_mat[ids[e]], c_e = c_mat[ids[e]] (uint8 ids, torch or numpy)."""
    n = len(k_mat)
    if len(c_mat) != n:
        raise HfError(HF_E_ARG, "k_mat and c_mat differ in length")
    ptr = None
    try:
        import torch
        if isinstance(ids, torch.Tensor):
            if ids.dtype != torch.uint8 or not ids.is_contiguous() or ids.numel() != ctx.n_elems:
                raise HfError(HF_E_ARG, "ids: need a contiguous uint8 tensor of n_elements")
            if ids.is_cuda and ids.device.index != ctx.device:
                raise HfError(HF_E_ARG, f"ids: tensor on {ids.device}, context on cuda:{ctx.device}")
            ptr = ids.data_ptr()
    except ImportError:
        pass
    if ptr is None:
        import numpy as np
        if not isinstance(ids, np.ndarray) or ids.dtype != np.uint8 or not ids.flags.c_contiguous \
                or ids.size != ctx.n_elems:
            raise HfError(HF_E_ARG, "ids: need a contiguous uint8 array of n_elements")
        ptr = ids.ctypes.data
    km = (C.c_double * n)(*[float(v) for v in k_mat])
    cm = (C.c_double * n)(*[float(v) for v in c_mat])
    _check(_lib.hf_set_material_ids(ctx.ptr, C.c_void_p(ptr), n, km, cm))


def hf_apply_impl(ctx: Context, impl: int, aK: float, aM: float, c: float, u, b, y):
    """NEXT f4 ablation: Implementation 1 (two-pass, stored element matrices), 2 (single-pass
    gather) or 3 (the production stencil) of the same apply."""
    _check(_lib.hf_apply_impl(ctx.ptr, int(impl), aK, aM, c, _cptr(ctx, u, ctx.n_nodes, "u"),
                              _cptr(ctx, b, ctx.n_nodes, "b", allow_none=True), _cptr(ctx, y, ctx.n_nodes, "y")))


def hf_ablation_prepare(ctx: Context, aK: float, aM: float):
    _check(_lib.hf_ablation_prepare(ctx.ptr, aK, aM))


def hf_diag(ctx: Context, aK: float, aM: float, diag):
    _check(_lib.hf_diag(ctx.ptr, aK, aM, _cptr(ctx, diag, ctx.n_nodes, "diag")))


def hf_cg(ctx: Context, aK: float, aM: float, b, x, rtol=1e-12, max_iter=10000, replace_every=-1,
          raise_on_noconv: bool = True) -> dict:
    info = hf_cg_info()
    o = _opts(rtol, max_iter, replace_every)
    st = _lib.hf_cg(ctx.ptr, aK, aM, _cptr(ctx, b, ctx.n_nodes, "b"), _cptr(ctx, x, ctx.n_nodes, "x"), C.byref(o), C.byref(info))
    res = {"iters": info.iters, "status": info.status, "relres": info.relres, "delta": info.delta}
    if st != HF_OK and (raise_on_noconv or st not in (HF_E_NOCONV, HF_E_BREAKDOWN)):
        _check(st)
    res["rc"] = st
    return res


def _stats(s: hf_sim_stats) -> dict:
    return {"steps_done": s.steps_done, "total_iters": s.total_iters, "max_iters_step": s.max_iters_step,
            "first_failed_step": s.first_failed_step, "ms_total": s.ms_total, "ms_steps": s.ms_steps}


def hf_simulate(ctx: Context, theta: float, dt: float, nsteps: int, F, u, snap_plane: int = -1, snap=None,
                rtol=1e-12, max_iter=10000, replace_every=-1, raise_on_noconv: bool = True) -> dict:
    s = hf_sim_stats()
    o = _opts(rtol, max_iter, replace_every)
    st = _lib.hf_simulate(ctx.ptr, theta, dt, nsteps, _cptr(ctx, F, ctx.n_nodes, "F", allow_none=True),
                          _cptr(ctx, u, ctx.n_nodes, "u"), snap_plane,
                          _cptr(ctx, snap, nsteps * ctx.n_plane, "snap", allow_none=True), C.byref(o), C.byref(s))
    res = _stats(s)
    if st != HF_OK and (raise_on_noconv or st not in (HF_E_NOCONV, HF_E_BREAKDOWN)):
        _check(st)
    res["rc"] = st
    return res


def hf_simulate_resume(ctx: Context, theta: float, dt: float, nsteps: int, F, u, u_prev, step0: int,
                       rtol=1e-12, max_iter=10000, replace_every=-1) -> dict:
    s = hf_sim_stats()
    o = _opts(rtol, max_iter, replace_every)
    _check(_lib.hf_simulate_resume(ctx.ptr, theta, dt, nsteps, _cptr(ctx, F, ctx.n_nodes, "F", allow_none=True),
                                   _cptr(ctx, u, ctx.n_nodes, "u"), _cptr(ctx, u_prev, ctx.n_nodes, "u_prev", allow_none=True),
                                   step0, C.byref(o), C.byref(s)))
    return _stats(s)


def hf_simulate_batched(ctx: Context, B: int, k_batch, c_batch, theta: float, dt: float, nsteps: int, F, u_batch,
                        snap_plane: int = -1, front_out=None, rtol=1e-12, max_iter=10000, replace_every=-1) -> list:
    stats = (hf_sim_stats * max(B, 1))()
    o = _opts(rtol, max_iter, replace_every)
    _check(_lib.hf_simulate_batched(ctx.ptr, B, _cptr(ctx, k_batch, B * ctx.n_elems, "k_batch"),
                                    _cptr(ctx, c_batch, B * ctx.n_elems, "c_batch", allow_none=True), theta, dt, nsteps,
                                    _cptr(ctx, F, ctx.n_nodes, "F", allow_none=True),
                                    _cptr(ctx, u_batch, B * ctx.n_nodes, "u_batch"), snap_plane,
                                    _cptr(ctx, front_out, B * ctx.n_plane, "front_out", allow_none=True), C.byref(o), stats))
    return [_stats(stats[j]) for j in range(B)]


def hf_slab_plan(nz1: int, rank: int, nranks: int):
    lo, hi = C.c_int64(), C.c_int64()
    _check(_lib.hf_slab_plan(nz1, rank, nranks, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def hf_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib.hf_nccl_unique_id(buf))
    return buf.raw


def hf_local_group_create(nranks: int):
    out = C.c_void_p()
    _check(_lib.hf_local_group_create(nranks, C.byref(out)))
    return out


def hf_local_group_destroy(grp):
    _lib.hf_local_group_destroy(grp)


HF_PEER_BLOB_BYTES = 256
TRANSPORT_NCCL, TRANSPORT_PEER_LOCAL, TRANSPORT_PEER_IPC = 0, 1, 2


def hf_create_slab(grid, rank: int, nranks: int, uid=None, transport: int = TRANSPORT_PEER_IPC, device: int = 0,
                   stream=None) -> Context:
    """uid: 128 NCCL id bytes (transport 0), the hf_local_group handle (transport 1), or None
    (transport 2: then hf_peer_export / all-gather / hf_peer_connect, see hf_peer_setup)."""
    g = make_grid(grid)
    out = C.c_void_p()
    keep = None
    if transport == TRANSPORT_NCCL:
        keep = C.create_string_buffer(bytes(uid), 128)
        idp = C.cast(keep, C.c_void_p)
    else:
        idp = uid
    _check(_lib.hf_create_slab(C.byref(g), rank, nranks, idp, transport, device, _stream(stream, device),
                               C.byref(out)))
    lo, hi, lp, z0 = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(_lib.hf_slab_range(out, C.byref(lo), C.byref(hi), C.byref(lp), C.byref(z0)))
    ctx = Context(out.value, g, device, lp.value)
    ctx.slab = (lo.value, hi.value, lp.value, z0.value)
    return ctx


def hf_peer_export(ctx: Context) -> bytes:
    buf = C.create_string_buffer(HF_PEER_BLOB_BYTES)
    _check(_lib.hf_peer_export(ctx.ptr, buf))
    return buf.raw


def hf_peer_connect(ctx: Context, blobs: Sequence[bytes]):
    data = b"".join(bytes(b) for b in blobs)
    if any(len(b) != HF_PEER_BLOB_BYTES for b in blobs):
        raise HfError(HF_E_ARG, "peer blobs must be HF_PEER_BLOB_BYTES each")
    _check(_lib.hf_peer_connect(ctx.ptr, data))


def hf_peer_setup(ctx: Context, all_gather):
    """Transport 2 handshake: all_gather(bytes) -> list of every rank's bytes in rank order
    (e.g. torch.distributed.all_gather_object); marshalling only."""
    hf_peer_connect(ctx, all_gather(hf_peer_export(ctx)))


def hf_slab_range(ctx: Context):
    lo, hi, lp, z0 = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    _check(_lib.hf_slab_range(ctx.ptr, C.byref(lo), C.byref(hi), C.byref(lp), C.byref(z0)))
    return lo.value, hi.value, lp.value, z0.value


def hf_get_launch_count(ctx: Context) -> int:
    v = C.c_int64()
    _check(_lib.hf_get_launch_count(ctx.ptr, C.byref(v)))
    return v.value


def hf_profile(ctx: Context, enable: bool):
    _check(_lib.hf_profile(ctx.ptr, 1 if enable else 0))


def hf_profile_read(ctx: Context):
    ms = (C.c_double * 5)()
    n = (C.c_int64 * 5)()
    _check(_lib.hf_profile_read(ctx.ptr, C.byref(ms), C.byref(n)))
    names = ["stencil_cg_a", "pointwise_cg_b", "residual", "rhs_apply", "other"]
    return {nm: (ms[i], n[i]) for i, nm in enumerate(names)}


def hf_set_driver(ctx: Context, driver: int):
    _check(_lib.hf_set_driver(ctx.ptr, driver))


def hf_set_mixed(ctx: Context, enable: int, rtol_lo: float = 1e-6):
    _check(_lib.hf_set_mixed(ctx.ptr, enable, rtol_lo))


def hf_mixed_iters(ctx: Context) -> int:
    v = C.c_int64()
    _check(_lib.hf_mixed_iters(ctx.ptr, C.byref(v)))
    return int(v.value)


def hf_set_tuning(ctx: Context, key: str, value: int):
    """Performance knob of the context (see heatfem.h: tile_r, zchunk, unroll, pdl, fuse_ab,
    check_every, tm_fence, batch_group, comm_timeout_s)."""
    _check(_lib.hf_set_tuning(ctx.ptr, key.encode(), int(value)))


def hf_get_tuning(ctx: Context, key: str) -> int:
    v = C.c_int64()
    _check(_lib.hf_get_tuning(ctx.ptr, key.encode(), C.byref(v)))
    return int(v.value)


def hf_set_cg_variant(ctx: Context, variant: int):
    _check(_lib.hf_set_cg_variant(ctx.ptr, variant))


def hf_cg_variant(ctx: Context) -> dict:
    out = (C.c_int32 * 2)()
    _check(_lib.hf_cg_variant(ctx.ptr, out))
    return {"variant": int(out[0]), "last_used": int(out[1])}


def hf_set_resident(ctx: Context, mode: int):
    _check(_lib.hf_set_resident(ctx.ptr, mode))


def hf_resident_plan(ctx: Context) -> dict:
    out = (C.c_int32 * 10)()
    _check(_lib.hf_resident_plan(ctx.ptr, out))
    keys = ("eligible", "px", "py", "pz", "bx", "by", "bz", "BZ", "smem_kb", "last_used")
    d = {k: int(v) for k, v in zip(keys, out)}
    if not d["eligible"]:
        d["why"] = _lib.hf_last_error().decode()
    return d


def hf_resident_profile(ctx: Context, enable: int) -> dict:
    out = (C.c_double * 24)()
    _check(_lib.hf_resident_profile(ctx.ptr, enable, out))
    keys = ("d_update_us", "stencil_us", "reduce_dq_us", "kernel_b_us", "reduce_rs_us", "init_us", "iters",
            "fence_us", "spin_us", "read_us")
    d = {k: float(v) for k, v in zip(keys, out[:10])}
    d.update({"max_" + k: float(v) for k, v in zip(keys, out[12:22])})
    return d


def hf_flush_l2(ctx: Context):
    _check(_lib.hf_flush_l2(ctx.ptr))


def hf_time_kernel_a(ctx: Context, reps: int = 200) -> float:
    """ms per launch of PCG kernel A replayed back to back (instrumentation, see heatfem.h)."""
    ms = C.c_double()
    _check(_lib.hf_time_kernel_a(ctx.ptr, reps, C.byref(ms)))
    return ms.value


def hf_time_kernel_a_graph(ctx: Context, reps: int = 200) -> float:
    """ms per launch of PCG kernel A replayed as a graph chain with the loop's programmatic edges."""
    ms = C.c_double()
    _check(_lib.hf_time_kernel_a_graph(ctx.ptr, reps, C.byref(ms)))
    return ms.value


def hf_set_precision(ctx: Context, bits: int):
    """64 (default) or 32: storage precision of the context (fp32 variant, NEXT row f3)."""
    _check(_lib.hf_set_precision(ctx.ptr, bits))


def hf_set_element(ctx: Context, elem_type: int):
    """0: trilinear hexahedra (default); 1: the paper's 6 P1 tets per voxel."""
    _check(_lib.hf_set_element(ctx.ptr, elem_type))


def hf_set_step_flush(ctx: Context, enable: bool):
    _check(_lib.hf_set_step_flush(ctx.ptr, 1 if enable else 0))


LIB_PATH = _LIB_PATH
