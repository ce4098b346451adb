"""Python binding of the libig C ABI: same names as include/ig.h, torch tensors in, pointers out.

Only argument marshalling happens here: every step of the hot path runs in libig's CUDA
kernels.  torch supplies device memory, the current stream and process groups.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import (  # noqa: F401
    IG_E_ARG,
    IG_EXTRAP_LS,
    IG_EXTRAP_SPARSE,
    IG_MAX_HISTORY,
    IG_OK,
    IG_PROJ_CLASSIC,
    IG_PROJ_QR,
    STATUS_NAMES,
    ig_stats_t,
    lib,
)

METHODS = {"proj_qr": IG_PROJ_QR, "extrap_ls": IG_EXTRAP_LS, "proj_classic": IG_PROJ_CLASSIC,
           "extrap_sparse": IG_EXTRAP_SPARSE}


class IGError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().ig_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _check(rc: int, where: str) -> None:
    if rc != IG_OK:
        raise IGError(rc, where)


def _dptr(t, name: str, N: int | None = None):
    """Device pointer of a contiguous fp64 CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CUDA tensor")
    if N is not None and t.numel() != N:
        raise ValueError(f"{name} has {t.numel()} elements, expected {N}")
    return t.data_ptr()


def _hptr(t, name: str, N: int | None = None):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or t.dtype != torch.float64 or t.is_cuda or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous float64 CPU tensor")
    if N is not None and t.numel() != N:
        raise ValueError(f"{name} has {t.numel()} elements, expected {N}")
    return t.data_ptr()


# ------------------------------------------------------------------ C-ABI mirrors
def ig_create(N: int, method: int, m: int, degree: int = 0, stream=None):
    h = lib().ig_create(int(N), int(method), int(m), int(degree))
    if not h:
        raise IGError(IG_E_ARG, "ig_create")
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().ig_set_stream(h, C.c_void_p(s.cuda_stream)), "ig_set_stream")
    return h


def ig_storage_bytes(N: int, method: int, m: int) -> int:
    return int(lib().ig_storage_bytes(int(N), int(method), int(m)))


def ig_create_ext(N: int, method: int, m: int, degree: int, storage, stream=None):
    """Handle whose history slabs live in caller-owned device memory (e.g. a torch uint8/fp64 tensor)."""
    if not isinstance(storage, torch.Tensor) or not storage.is_cuda or not storage.is_contiguous():
        raise TypeError("storage must be a contiguous CUDA tensor")
    nbytes = storage.numel() * storage.element_size()
    h = lib().ig_create_ext(int(N), int(method), int(m), int(degree), C.c_void_p(storage.data_ptr()), nbytes)
    if not h:
        raise IGError(IG_E_ARG, "ig_create_ext")
    s = stream if stream is not None else torch.cuda.current_stream()
    _check(lib().ig_set_stream(h, C.c_void_p(s.cuda_stream)), "ig_set_stream")
    return h


def ig_destroy(h) -> None:
    lib().ig_destroy(h)


def ig_reset(h) -> None:
    _check(lib().ig_reset(h), "ig_reset")


def ig_set_admit_tol(h, eps: float) -> None:
    _check(lib().ig_set_admit_tol(h, float(eps)), "ig_set_admit_tol")


def ig_set_schedule(h, fused: bool) -> None:
    _check(lib().ig_set_schedule(h, 1 if fused else 0), "ig_set_schedule")


def ig_set_stream(h, stream) -> None:
    _check(lib().ig_set_stream(h, C.c_void_p(stream.cuda_stream)), "ig_set_stream")


def ig_form_guess(h, b, x0) -> None:
    _check(lib().ig_form_guess(h, _dptr(b, "b"), _dptr(x0, "x0")), "ig_form_guess")


def ig_update(h, x, Ax=None) -> None:
    _check(lib().ig_update(h, _dptr(x, "x"), _dptr(Ax, "Ax")), "ig_update")


def _ptr_array(vals):
    return (C.c_void_p * len(vals))(*[C.c_void_p(v) if v else None for v in vals])


def ig_form_guess_batch(handles, bs, x0s) -> None:
    """Guesses of several fields; consecutive extrapolation fields share one kernel launch."""
    n = len(handles)
    hb = _ptr_array([h.h if isinstance(h, InitialGuess) else h for h in handles])
    bp = _ptr_array([_dptr(b, "b") for b in bs]) if bs is not None else None
    xp = _ptr_array([_dptr(x, "x0") for x in x0s])
    _check(lib().ig_form_guess_batch(n, hb, bp, xp), "ig_form_guess_batch")


def ig_update_batch(handles, xs, Axs=None) -> None:
    n = len(handles)
    hb = _ptr_array([h.h if isinstance(h, InitialGuess) else h for h in handles])
    xp = _ptr_array([_dptr(x, "x") for x in xs])
    ap = _ptr_array([_dptr(a, "Ax") for a in Axs]) if Axs is not None else None
    _check(lib().ig_update_batch(n, hb, xp, ap), "ig_update_batch")


def ig_form_guess_batch_host(handles, bs, x0s) -> None:
    """Host-buffer batch guess (include/ig.h): transfers of the fields overlap; syncs once."""
    n = len(handles)
    hb = _ptr_array([h.h if isinstance(h, InitialGuess) else h for h in handles])
    bp = _ptr_array([_hptr(b, "b") for b in bs]) if bs is not None else None
    xp = _ptr_array([_hptr(x, "x0") for x in x0s])
    _check(lib().ig_form_guess_batch_host(n, hb, bp, xp), "ig_form_guess_batch_host")


def ig_update_batch_host(handles, xs, Axs=None) -> None:
    n = len(handles)
    hb = _ptr_array([h.h if isinstance(h, InitialGuess) else h for h in handles])
    xp = _ptr_array([_hptr(x, "x") for x in xs])
    ap = _ptr_array([_hptr(a, "Ax") for a in Axs]) if Axs is not None else None
    _check(lib().ig_update_batch_host(n, hb, xp, ap), "ig_update_batch_host")


def ig_form_guess_host(h, b, x0) -> None:
    _check(lib().ig_form_guess_host(h, _hptr(b, "b"), _hptr(x0, "x0")), "ig_form_guess_host")


def ig_update_host(h, x, Ax=None) -> None:
    _check(lib().ig_update_host(h, _hptr(x, "x"), _hptr(Ax, "Ax")), "ig_update_host")


def ig_next_slot(h) -> int:
    """Device address of the extrapolation zero-copy slot (0 for projection handles)."""
    return lib().ig_next_slot(h) or 0


def ig_history_dim(h) -> int:
    d = C.c_int()
    _check(lib().ig_history_dim(h, C.byref(d)), "ig_history_dim")
    return d.value


def ig_weights(h, f: int = 0):
    beta = (C.c_double * IG_MAX_HISTORY)()
    n = C.c_int()
    _check(lib().ig_weights(h, int(f), beta, C.byref(n)), "ig_weights")
    return [beta[i] for i in range(n.value)]


def ig_bytes(h):
    fb, ub = C.c_int64(), C.c_int64()
    _check(lib().ig_bytes(h, C.byref(fb), C.byref(ub)), "ig_bytes")
    return fb.value, ub.value


def ig_get_stats(h) -> dict:
    s = ig_stats_t()
    _check(lib().ig_get_stats(h, C.byref(s)), "ig_get_stats")
    return {k: getattr(s, k) for k, _ in ig_stats_t._fields_}


def ig_copy_history(h, M: int, N: int):
    """(Bt[M,N], Xt[M,N]) device copies and R[M,M] (host) of a projection handle."""
    Bt = torch.empty((M, N), dtype=torch.float64, device="cuda")
    Xt = torch.empty((M, N), dtype=torch.float64, device="cuda")
    R = (C.c_double * (M * M))()
    _check(lib().ig_copy_history(h, Bt.data_ptr(), Xt.data_ptr(), N, R), "ig_copy_history")
    Rt = torch.tensor(list(R), dtype=torch.float64).reshape(M, M).T.contiguous()  # column-major -> [i, j]
    return Bt, Xt, Rt


def ig_total_launches() -> int:
    return int(lib().ig_total_launches())


def ig_profile(h, enable: bool) -> None:
    _check(lib().ig_profile(h, 1 if enable else 0), "ig_profile")


def ig_profile_read(h) -> dict:
    """{kernel name: (total_ms, launches)} since the last ig_profile call (syncs)."""
    from ._lib import KERNELS

    out = {}
    for k, name in enumerate(KERNELS):
        ms, n = C.c_double(), C.c_int64()
        _check(lib().ig_profile_read(h, k, C.byref(ms), C.byref(n)), "ig_profile_read")
        out[name] = (ms.value, n.value)
    return out


def ig_comm_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    _check(lib().ig_comm_unique_id(buf), "ig_comm_unique_id")
    return bytes(buf)


def ig_comm_create(nranks: int, rank: int, uid: bytes):
    if len(uid) != 128:
        raise ValueError("unique id must be 128 bytes")
    out = C.c_void_p()
    _check(lib().ig_comm_create(int(nranks), int(rank), C.c_char_p(uid), C.byref(out)), "ig_comm_create")
    return out.value


def ig_comm_destroy(c) -> None:
    lib().ig_comm_destroy(c)


def ig_local_group_create(nranks: int):
    """In-process rank group (include/ig.h): ranks are threads of this process."""
    g = lib().ig_local_group_create(int(nranks))
    if not g:
        raise IGError(IG_E_ARG, "ig_local_group_create")
    return g


def ig_local_group_destroy(g) -> None:
    lib().ig_local_group_destroy(g)


def ig_comm_create_local(group, rank: int):
    out = C.c_void_p()
    _check(lib().ig_comm_create_local(group, int(rank), C.byref(out)), "ig_comm_create_local")
    return out.value


def ig_attach_comm(h, c) -> None:
    _check(lib().ig_attach_comm(h, c), "ig_attach_comm")


def _nccl_path() -> str | None:
    try:
        import nvidia.nccl

        for p in nvidia.nccl.__path__:
            cand = os.path.join(p, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand
    except ImportError:
        pass
    return None


def comm_from_process_group(group=None):
    """NCCL communicator for libig over the ranks of a torch.distributed group.

    Rank 0 draws the NCCL unique id through libig; torch.distributed broadcasts the 128 bytes
    (plumbing only).  Every rank must use its own GPU (torch.cuda.set_device before this).
    """
    import torch.distributed as dist

    if "IG_NCCL_PATH" not in os.environ:
        p = _nccl_path()
        if p:
            os.environ["IG_NCCL_PATH"] = p
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [ig_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return ig_comm_create(world, rank, obj[0])


def ig_save_state(h) -> bytes:
    """Checkpoint image of one history space (host bytes)."""
    n = int(lib().ig_state_bytes(h))
    buf = (C.c_char * n)()
    _check(lib().ig_save_state(h, buf, n), "ig_save_state")
    return bytes(buf)


def ig_load_state(h, image: bytes) -> None:
    _check(lib().ig_load_state(h, C.c_char_p(image), len(image)), "ig_load_state")


def ig_set_grid_limit(h, max_blocks: int) -> None:
    _check(lib().ig_set_grid_limit(h, int(max_blocks)), "ig_set_grid_limit")


def ig_set_launch(h, cooperative: int) -> None:
    """Persistent kernels: 1 cooperative (default), 0 plain launch, -1 process default (ig.h)."""
    _check(lib().ig_set_launch(h, int(cooperative)), "ig_set_launch")


def ig_set_device_ring(h, on: bool) -> None:
    """Extrapolation window position in device memory: graph-capturable form / push (ig.h)."""
    _check(lib().ig_set_device_ring(h, 1 if on else 0), "ig_set_device_ring")


def ig_capture_begin(stream) -> None:
    _check(lib().ig_capture_begin(C.c_void_p(stream.cuda_stream)), "ig_capture_begin")


def ig_capture_end(stream):
    out = C.c_void_p()
    _check(lib().ig_capture_end(C.c_void_p(stream.cuda_stream), C.byref(out)), "ig_capture_end")
    return out.value


def ig_graph_launch(g, stream) -> None:
    _check(lib().ig_graph_launch(g, C.c_void_p(stream.cuda_stream)), "ig_graph_launch")


def ig_graph_destroy(g) -> None:
    lib().ig_graph_destroy(g)


class CapturedStep:
    """`with CapturedStep(stream) as step:` captures the libig calls issued on `stream` (every
    handle set to it) into a CUDA graph; `step.replay()` relaunches it (ig_capture_* in ig.h)."""

    def __init__(self, stream):
        self.stream, self.g = stream, None

    def __enter__(self):
        ig_capture_begin(self.stream)
        return self

    def __exit__(self, exc_type, exc, tb):
        if exc_type is not None:  # end the capture, drop the partial graph
            try:
                ig_graph_destroy(ig_capture_end(self.stream))
            except IGError:
                pass
            return False
        self.g = ig_capture_end(self.stream)
        return False

    def replay(self) -> None:
        ig_graph_launch(self.g, self.stream)

    def close(self) -> None:
        if self.g:
            ig_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ig_set_watchdog(h, seconds: float) -> None:
    _check(lib().ig_set_watchdog(h, float(seconds)), "ig_set_watchdog")


def ig_xwin_export(h) -> bytes:
    buf = (C.c_char * 64)()
    _check(lib().ig_xwin_export(h, buf), "ig_xwin_export")
    return bytes(buf)


def ig_xwin_ptr(h) -> int:
    p = lib().ig_xwin_ptr(h)
    if not p:
        raise IGError(IG_E_ARG, "ig_xwin_ptr")
    return p


def ig_attach_peers(h, nranks: int, rank: int, ipc_handles: bytes | None = None, peer_ptrs=None) -> None:
    ptrs = None
    if peer_ptrs is not None:
        ptrs = (C.c_void_p * nranks)(*[C.c_void_p(p) if p else None for p in peer_ptrs])
    hb = C.c_char_p(ipc_handles) if ipc_handles is not None else None
    _check(lib().ig_attach_peers(h, int(nranks), int(rank), hb, ptrs), "ig_attach_peers")


def peers_from_process_group(handles, group=None) -> None:
    """Collective: wire the in-kernel NVLink peer exchange of `handles` (one per field, same order
    on every rank) across the ranks of a torch.distributed group (IPC handles travel through
    torch.distributed; plumbing only)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device()
    devs = [None] * world
    dist.all_gather_object(devs, (socket_host(), dev), group=group)
    why = None
    for host, d in devs:
        if host != socket_host():
            why = "the in-kernel peer exchange needs all ranks on one node"
        elif d != dev and not torch.cuda.can_device_access_peer(dev, d):
            why = f"GPU {dev} cannot access GPU {d} (no P2P/NVLink)"
    verdicts = [None] * world
    dist.all_gather_object(verdicts, why, group=group)  # every rank takes the same decision
    bad = [v for v in verdicts if v]
    if bad:
        raise RuntimeError(bad[0] + ": use the NCCL exchange")
    for h in handles:
        mine = ig_xwin_export(h)
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        ig_attach_peers(h, world, rank, b"".join(allh))
    dist.barrier(group=group)


def socket_host() -> str:
    import socket

    return socket.gethostname()


def attach_virtual_ranks(handles) -> None:
    """Wire handles living in ONE process on ONE GPU as ranks of an in-kernel exchange (tests)."""
    ptrs = [ig_xwin_ptr(h) for h in handles]
    for r, h in enumerate(handles):
        ig_attach_peers(h, len(handles), r, None, ptrs)


def shard_range(N_total: int, world: int, rank: int):
    """Contiguous DOF range [lo, hi) of `rank` (z-slab partition); sizes differ by <= 1."""
    base, rem = divmod(int(N_total), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


# ------------------------------------------------------------------ convenience object
class InitialGuess:
    """One history space (one field).  Thin wrapper over an ig_t handle."""

    def __init__(self, N: int, method="proj_qr", m: int = 8, degree: int = 0, eps: float | None = None,
                 comm=None, stream=None, fused: bool = True, storage=None):
        self.N, self.m, self.degree = int(N), int(m), int(degree)
        self.method = METHODS[method] if isinstance(method, str) else int(method)
        self.storage = storage  # keep caller-provided history memory alive with the handle
        if storage is None:
            self.h = ig_create(self.N, self.method, self.m, self.degree, stream)
        else:
            self.h = ig_create_ext(self.N, self.method, self.m, self.degree, storage, stream)
        if eps is not None:
            ig_set_admit_tol(self.h, eps)
        if not fused:
            ig_set_schedule(self.h, False)
        if comm is not None:
            ig_attach_comm(self.h, comm)

    def form_guess(self, b, x0):
        ig_form_guess(self.h, b, x0)
        return x0

    def update(self, x, Ax=None):
        ig_update(self.h, x, Ax)

    def set_device_ring(self, on: bool = True) -> None:
        ig_set_device_ring(self.h, on)

    def set_stream(self, stream) -> None:
        ig_set_stream(self.h, stream)

    def next_slot(self):
        """torch view of the extrapolation zero-copy slot."""
        addr = ig_next_slot(self.h)
        if not addr:
            return None
        return _view(addr, self.N)

    @property
    def d(self) -> int:
        return ig_history_dim(self.h)

    def stats(self) -> dict:
        return ig_get_stats(self.h)

    def bytes(self):
        return ig_bytes(self.h)

    def weights(self, f: int = 0):
        return ig_weights(self.h, f)

    def save_state(self) -> bytes:
        return ig_save_state(self.h)

    def load_state(self, image: bytes) -> None:
        ig_load_state(self.h, image)

    def reset(self):
        ig_reset(self.h)

    def close(self):
        if self.h:
            ig_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _CAI:
    def __init__(self, addr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (addr, False), "version": 3,
                                         "strides": None}


def _view(addr: int, n: int) -> torch.Tensor:
    """Zero-copy torch view of library-owned device memory (CUDA array interface)."""
    return torch.as_tensor(_CAI(addr, n), device="cuda")
