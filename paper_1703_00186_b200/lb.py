"""Thin Python binding of the C ABI in include/lb.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of liblb_d2q37.so; this
module allocates the two population buffers as torch tensors, passes their
device pointers and the current torch stream, and maps status codes to
exceptions.  There is no CPU fallback: if the library is missing or there is
no CUDA device, construction raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

Q = 37
HALO = 3
STATUS = {0: "LB_OK", 1: "LB_EINVAL", 2: "LB_ESTATE", 3: "LB_ECUDA", 4: "LB_ENCCL",
          5: "LB_ENONPHYS", 6: "LB_ENOMEM", 7: "LB_EPEER"}
BC = {"thermal": 0, "adiabatic": 1, "periodic": 2}
MODE = {"fused": 0, "split": 1}
COLLISION = {"bgk": 0, "regularized": 1}

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "liblb_d2q37.so")

# every symbol include/lb.h declares
EXPORTS = ["lb_query_layout", "lb_exchange_plan", "lb_constants", "lb_kwall", "lb_nccl_unique_id", "lb_last_error",
           "lb_strerror", "lb_init", "lb_destroy", "lb_get_layout", "lb_set_stream", "lb_init_macro", "lb_init_rt",
           "lb_set_state", "lb_exchange", "lb_propagate", "lb_bc", "lb_collide", "lb_step",
           "lb_gather", "lb_peek", "lb_invariants", "lb_sync", "lb_profile_enable",
           "lb_profile_reset", "lb_profile_read", "lb_launch_count", "lb_tb_strip_height", "lb_set_peers",
           "lb_monitor", "lb_peek_cols", "lb_set_option", "lb_invariants_async", "lb_invariants_pair_async"]


class LBError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class lb_params(ctypes.Structure):
    _fields_ = [("lx_total", ctypes.c_int), ("ly", ctypes.c_int), ("tau", ctypes.c_double),
                ("dt", ctypes.c_double), ("t_bottom", ctypes.c_double), ("t_top", ctypes.c_double),
                ("bc_y", ctypes.c_int), ("mode", ctypes.c_int), ("overlap", ctypes.c_int),
                ("collision", ctypes.c_int), ("gx", ctypes.c_double), ("gy", ctypes.c_double)]


class lb_dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_id", ctypes.c_void_p)]


class lb_layout(ctypes.Structure):
    _fields_ = [("lx", ctypes.c_int), ("ly", ctypes.c_int), ("nx", ctypes.c_int), ("nyp", ctypes.c_int),
                ("y0", ctypes.c_int), ("x0_global", ctypes.c_int), ("col_stride", ctypes.c_int64),
                ("elems", ctypes.c_int64), ("bytes", ctypes.c_int64), ("sites", ctypes.c_int64)]


class lb_xplan(ctypes.Structure):
    _fields_ = [("left", ctypes.c_int), ("right", ctypes.c_int), ("count", ctypes.c_int64),
                ("recv_left_off", ctypes.c_int64), ("recv_right_off", ctypes.c_int64),
                ("send_right_off", ctypes.c_int64), ("send_left_off", ctypes.c_int64),
                ("bulk_x0", ctypes.c_int), ("bulk_x1", ctypes.c_int),
                ("border_x0", ctypes.c_int), ("border_x1", ctypes.c_int),
                ("border_x2", ctypes.c_int), ("border_x3", ctypes.c_int)]


class lb_peers(ctypes.Structure):
    _fields_ = [("left_buf", ctypes.c_void_p * 2), ("right_buf", ctypes.c_void_p * 2),
                ("left_done", ctypes.c_void_p), ("right_done", ctypes.c_void_p),
                ("my_done", ctypes.c_void_p)]


class lb_kprof(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_int64),
                ("total_ms", ctypes.c_double), ("units", ctypes.c_int64)]


_lib = None


def lib():
    """Load liblb_d2q37.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    import torch  # noqa: F401  (loads the wheel's libnccl.so.2 / CUDA runtime first)
    from . import _build
    alt = os.environ.get("LB_D2Q37_LIB")  # tools only: a variant build of the same sources
    if alt:
        L = ctypes.CDLL(alt)
    else:
        if _build.needs_build():
            _build.build()
        L = ctypes.CDLL(SO_PATH)
    p, i, d, vp = ctypes.POINTER, ctypes.c_int, ctypes.c_double, ctypes.c_void_p
    sig = {
        "lb_query_layout": (i, [p(lb_params), i, i, p(lb_layout)]),
        "lb_constants": (i, [vp, vp, vp, vp]),
        "lb_exchange_plan": (i, [p(lb_params), i, i, p(lb_xplan)]),
        "lb_kwall": (i, [d, vp]),
        "lb_nccl_unique_id": (i, [vp]),
        "lb_last_error": (ctypes.c_char_p, []),
        "lb_strerror": (ctypes.c_char_p, [i]),
        "lb_init": (i, [p(lb_params), p(lb_dist), vp, vp, vp, p(vp)]),
        "lb_destroy": (None, [vp]),
        "lb_get_layout": (i, [vp, p(lb_layout)]),
        "lb_set_stream": (i, [vp, vp]),
        "lb_init_macro": (i, [vp, vp, vp, vp, vp, i]),
        "lb_init_rt": (i, [vp, vp, d, d, d]),
        "lb_set_state": (i, [vp, vp, i]),
        "lb_exchange": (i, [vp]), "lb_propagate": (i, [vp]), "lb_bc": (i, [vp]),
        "lb_collide": (i, [vp]), "lb_step": (i, [vp, i]),
        "lb_gather": (i, [vp, vp, i]),
        "lb_peek": (i, [vp, i, vp]),
        "lb_peek_cols": (i, [vp, i, i, i, vp]),
        "lb_invariants": (i, [vp, vp]),
        "lb_invariants_async": (i, [vp, vp]),
        "lb_invariants_pair_async": (i, [vp, vp]),
        "lb_sync": (i, [vp]),
        "lb_profile_enable": (i, [vp, i]), "lb_profile_reset": (i, [vp]),
        "lb_profile_read": (i, [vp, p(lb_kprof), i, p(i)]),
        "lb_launch_count": (ctypes.c_int64, [vp]),
        "lb_tb_strip_height": (i, []),
        "lb_set_peers": (i, [vp, p(lb_peers)]),
        "lb_monitor": (i, [vp, i]),
        "lb_set_option": (i, [vp, i, i]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise LBError(status, lib().lb_last_error().decode())


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


# ---- host-only helpers (no GPU needed) ----------------------------------------

def constants():
    """(c[37,2] int, w[37], a, T0) as the library uses them."""
    c = np.zeros(2 * Q, dtype=np.int32)
    w = np.zeros(Q)
    a = ctypes.c_double()
    t0 = ctypes.c_double()
    _check(lib().lb_constants(c.ctypes.data_as(ctypes.c_void_p), _dptr(w), ctypes.byref(a), ctypes.byref(t0)))
    return c.reshape(Q, 2).astype(np.int64), w, a.value, t0.value


def tb_strip_height() -> int:
    """Strip height HT of the library's two-step kernel (lb_tb_strip_height)."""
    return int(lib().lb_tb_strip_height())


def t0() -> float:
    return constants()[3]


def kwall(t_wall: float) -> np.ndarray:
    K = np.zeros(Q)
    _check(lib().lb_kwall(float(t_wall), _dptr(K)))
    return K


def make_params(lx_total, ly, tau=0.8, dt=1.0, t_bottom=None, t_top=None, bc_y="thermal",
                mode="fused", overlap=False, collision="bgk", gravity=(0.0, 0.0)) -> lb_params:
    T0 = t0()
    return lb_params(int(lx_total), int(ly), float(tau), float(dt),
                     float(1.05 * T0 if t_bottom is None else t_bottom),
                     float(0.95 * T0 if t_top is None else t_top),
                     BC[bc_y] if isinstance(bc_y, str) else int(bc_y),
                     MODE[mode] if isinstance(mode, str) else int(mode), int(bool(overlap)),
                     COLLISION[collision] if isinstance(collision, str) else int(collision),
                     float(gravity[0]), float(gravity[1]))


def query_layout(params: lb_params, rank: int = 0, nranks: int = 1) -> lb_layout:
    L = lb_layout()
    _check(lib().lb_query_layout(ctypes.byref(params), rank, nranks, ctypes.byref(L)))
    return L


def exchange_plan(params: lb_params, rank: int = 0, nranks: int = 1) -> lb_xplan:
    X = lb_xplan()
    _check(lib().lb_exchange_plan(ctypes.byref(params), rank, nranks, ctypes.byref(X)))
    return X


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().lb_nccl_unique_id(buf))
    return bytes(buf)


# ---- the lattice context --------------------------------------------------------

class Lattice:
    """One rank's X-slab of the D2Q37 lattice on the current CUDA device.

    Buffers A/B are torch float64 tensors owned by this object (the library
    borrows them, include/lb.h "Ownership")."""

    def __init__(self, lx_total, ly, tau=0.8, dt=1.0, t_bottom=None, t_top=None, bc_y="thermal",
                 mode="fused", overlap=False, rank=0, nranks=1, nccl_id: bytes | None = None,
                 device=None, stream=None, collision="bgk", gravity=(0.0, 0.0), temporal=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1703_00186_b200 needs a CUDA device (no CPU fallback)")
        self.params = make_params(lx_total, ly, tau, dt, t_bottom, t_top, bc_y, mode, overlap, collision,
                                  gravity)
        self.layout = query_layout(self.params, rank, nranks)
        self.rank, self.nranks = rank, nranks
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.stream = torch.cuda.current_stream(self.device) if stream is None else stream
        n = int(self.layout.elems)
        self.bufs = [torch.empty(n, dtype=torch.float64, device=self.device) for _ in range(2)]
        self._id = (ctypes.c_ubyte * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        dist = lb_dist(rank, nranks, ctypes.cast(self._id, ctypes.c_void_p) if self._id is not None else None)
        ctx = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib().lb_init(ctypes.byref(self.params), ctypes.byref(dist),
                                 ctypes.c_void_p(self.bufs[0].data_ptr()),
                                 ctypes.c_void_p(self.bufs[1].data_ptr()),
                                 ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(ctx)))
        self._ctx = ctx
        if temporal is not None:   # None: the library default (two-step kernel where it applies)
            _check(lib().lb_set_option(self._ctx, 3, int(bool(temporal))))

    # lifetime
    def close(self):
        if getattr(self, "_ctx", None):
            lib().lb_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def lx(self):
        return self.layout.lx

    @property
    def ly(self):
        return self.layout.ly

    @property
    def sites(self):
        return int(self.layout.sites)

    # state in
    def init_macro(self, rho, ux, uy, T):
        import torch
        arrs = [rho, ux, uy, T]
        if all(isinstance(a, torch.Tensor) and a.is_cuda for a in arrs):
            arrs = [a.contiguous() for a in arrs]
            for a in arrs:
                assert a.dtype == torch.float64 and a.numel() == self.sites
            _check(lib().lb_init_macro(self._ctx, *[ctypes.c_void_p(a.data_ptr()) for a in arrs], 1))
            self._keep = arrs
        else:
            arrs = [np.ascontiguousarray(np.asarray(a, dtype=np.float64)) for a in arrs]
            for a in arrs:
                assert a.size == self.sites
            _check(lib().lb_init_macro(self._ctx, *[_dptr(a) for a in arrs], 0))
            self.sync()

    def init_rt(self, eps, t_ref: float, amp: float = 0.05, width: float = 2.0):
        """Rayleigh-Taylor initial state evaluated on the device (lb_init_rt);
        eps: the lx_total column jitters (lbgen.rt_eps)."""
        e = np.ascontiguousarray(np.asarray(eps, dtype=np.float64))
        assert e.size == self.params.lx_total
        _check(lib().lb_init_rt(self._ctx, _dptr(e), float(t_ref), float(amp), float(width)))
        self.sync()

    def set_state(self, canon):
        import torch
        if isinstance(canon, torch.Tensor) and canon.is_cuda:
            assert canon.dtype == torch.float64 and canon.numel() == Q * self.sites
            canon = canon.contiguous()
            _check(lib().lb_set_state(self._ctx, ctypes.c_void_p(canon.data_ptr()), 1))
            self._keep = [canon]
        else:
            a = np.ascontiguousarray(np.asarray(canon, dtype=np.float64))
            assert a.size == Q * self.sites
            _check(lib().lb_set_state(self._ctx, _dptr(a), 0))
            self.sync()

    # the hot path
    def exchange(self):
        _check(lib().lb_exchange(self._ctx))

    def propagate(self):
        _check(lib().lb_propagate(self._ctx))

    def bc(self):
        _check(lib().lb_bc(self._ctx))

    def collide(self):
        _check(lib().lb_collide(self._ctx))

    def step(self, n: int = 1):
        _check(lib().lb_step(self._ctx, int(n)))

    def sync(self):
        _check(lib().lb_sync(self._ctx))

    # results
    def gather(self, root: int = 0, out: np.ndarray | None = None):
        """Canonical global state [37][lx_total][ly] on root (None elsewhere)."""
        shape = (Q, self.params.lx_total, self.ly)
        if self.rank == root:
            if out is None:
                out = np.empty(shape)
            assert out.shape == shape and out.dtype == np.float64 and out.flags.c_contiguous
            _check(lib().lb_gather(self._ctx, _dptr(out), root))
            return out
        _check(lib().lb_gather(self._ctx, None, root))
        return None

    def peek(self, which: int = 0) -> np.ndarray:
        out = np.empty((Q, self.lx, self.ly))
        _check(lib().lb_peek(self._ctx, which, _dptr(out)))
        return out

    def invariants_async(self, out) -> None:
        """Enqueue the invariants into `out` (5 float64, ideally a pinned torch
        tensor / its numpy view); valid after sync()."""
        import torch
        if isinstance(out, torch.Tensor):
            assert out.dtype == torch.float64 and out.numel() >= 5 and not out.is_cuda
            ptr = ctypes.c_void_p(out.data_ptr())
        else:
            ptr = _dptr(out)
        _check(lib().lb_invariants_async(self._ctx, ptr))

    def invariants_pair_async(self, out) -> None:
        """After a two-step lb_step(2) with monitors: enqueue the invariants of
        both states into `out` (10 float64: state n+1, then n+2); valid after sync()."""
        import torch
        if isinstance(out, torch.Tensor):
            assert out.dtype == torch.float64 and out.numel() >= 10 and not out.is_cuda and out.is_contiguous()
            ptr = ctypes.c_void_p(out.data_ptr())
        else:
            assert out.size >= 10 and out.dtype == np.float64
            ptr = _dptr(out)
        _check(lib().lb_invariants_pair_async(self._ctx, ptr))

    def peek_cols(self, x0: int, ncols: int, which: int = 0) -> np.ndarray:
        """Local physical columns [x0, x0+ncols) of A (0) or B (1): [37][ncols][ly]."""
        out = np.empty((Q, ncols, self.ly))
        _check(lib().lb_peek_cols(self._ctx, which, int(x0), int(ncols), _dptr(out)))
        return out

    def invariants(self) -> np.ndarray:
        """[sum rho, sum jx, sum jy, sum E, min rho] (raises LBError on LB_ENONPHYS)."""
        out = np.zeros(5)
        _check(lib().lb_invariants(self._ctx, _dptr(out)))
        return out

    # instrumentation
    def profile(self, enable: bool = True):
        _check(lib().lb_profile_enable(self._ctx, int(enable)))

    def profile_reset(self):
        _check(lib().lb_profile_reset(self._ctx))

    def profile_read(self) -> dict:
        recs = (lb_kprof * 64)()
        n = ctypes.c_int()
        _check(lib().lb_profile_read(self._ctx, recs, 64, ctypes.byref(n)))
        return {recs[i].name.decode(): {"launches": recs[i].launches, "total_ms": recs[i].total_ms,
                                        "units": recs[i].units} for i in range(min(n.value, 64))}

    def set_peers(self, left, right):
        """Peer-store exchange with neighbour lattices of THIS process (same
        device): left/right are Lattice objects (may be self).  Every rank must
        call it before any of them steps."""
        import torch
        if not hasattr(self, "done"):
            self.done = torch.zeros(1, dtype=torch.int64, device=self.device)
        for nb in (left, right):
            if not hasattr(nb, "done"):
                nb.done = torch.zeros(1, dtype=torch.int64, device=nb.device)
        P = lb_peers()
        P.left_buf[0], P.left_buf[1] = left.bufs[0].data_ptr(), left.bufs[1].data_ptr()
        P.right_buf[0], P.right_buf[1] = right.bufs[0].data_ptr(), right.bufs[1].data_ptr()
        P.left_done, P.right_done = left.done.data_ptr(), right.done.data_ptr()
        P.my_done = self.done.data_ptr()
        self._peers = (left, right)
        _check(lib().lb_set_peers(self._ctx, ctypes.byref(P)))

    def set_peers_ipc(self, group=None):
        """Peer-store exchange across processes (one rank per GPU, or several
        ranks sharing a GPU): every rank's buffers and step counter are shared
        with CUDA IPC (torch.multiprocessing's tensor reduction, which opens the
        handles with lazy peer access, i.e. NVLink P2P mappings), exchanged with
        torch.distributed.all_gather_object; then lb_set_peers and a barrier.
        Collective over the ring's process group."""
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor
        if not hasattr(self, "done"):
            self.done = torch.zeros(1, dtype=torch.int64, device=self.device)
        mine = [reduce_tensor(t) for t in (self.bufs[0], self.bufs[1], self.done)]
        allr = [None] * self.nranks
        dist.all_gather_object(allr, mine, group=group)
        left, right = (self.rank - 1) % self.nranks, (self.rank + 1) % self.nranks

        def open_rank(r):
            if r == self.rank:
                return [self.bufs[0], self.bufs[1], self.done]
            return [fn(*args) for fn, args in allr[r]]

        L, R = open_rank(left), open_rank(right)
        self._peer_tensors = (L, R)  # keep the IPC mappings alive
        self.set_peers_raw((L[0].data_ptr(), L[1].data_ptr()), (R[0].data_ptr(), R[1].data_ptr()),
                           L[2].data_ptr(), R[2].data_ptr(), self.done.data_ptr())
        dist.barrier(group=group)

    def set_peers_raw(self, left_bufs, right_bufs, left_done, right_done, my_done):
        """Peer-store exchange from raw device pointers (e.g. CUDA IPC mappings)."""
        P = lb_peers()
        P.left_buf[0], P.left_buf[1] = left_bufs
        P.right_buf[0], P.right_buf[1] = right_bufs
        P.left_done, P.right_done, P.my_done = left_done, right_done, my_done
        _check(lib().lb_set_peers(self._ctx, ctypes.byref(P)))

    def set_propagate_impl(self, impl: str):
        """'tma' (TMA-staged windows; the library default when the tensor maps
        encode, lb_init) or 'ldg' (register gather) for lb_propagate."""
        _check(lib().lb_set_option(self._ctx, 0, {"ldg": 0, "tma": 1}[impl]))

    def set_fused_impl(self, impl: str):
        """'ldg' (register gather, the default) or 'tma' (TMA-staged windows)
        for the one-step fused kernel (N=1, walls, monitors off)."""
        _check(lib().lb_set_option(self._ctx, 1, {"ldg": 0, "tma": 1}[impl]))

    def use_graphs(self, enable: bool = True):
        """Replay 2-step CUDA graphs in lb_step (needs a non-default stream)."""
        _check(lib().lb_set_option(self._ctx, 2, int(enable)))

    def temporal(self, enable: bool = True, grid: int = 0, l2_prefetch: int = 0, wall_weight16: int = 0,
                 l2_promotion: int | None = None, tail_weight16: int = 0, pdl: bool | None = None):
        """Two steps per pass over HBM (LB_OPT_TEMPORAL, the default where it
        applies: fused mode, walls, N = 1 or N > 1 in peer mode, monitors on or
        off — with monitors the kernel reduces both states' invariants):
        lb_step advances pairs of steps with the two-step kernel.  grid: CTAs
        (0 = one per SM); l2_prefetch: L2 prefetch distance in columns (0 = off);
        wall_weight16: cost of a wall-strip column, x16, for the work split
        (0 = the library default: 21 with the time-aligned split; contiguous: 19 BGK, 20 regularised);
        l2_promotion: L2 promotion of its TMA loads in bytes (None = library default);
        tail_weight16: cost of a tail-region column of the time-aligned split,
        x16 (0 = the library default: 17 with >= 2 main-region CTAs per strip, else 16;
        1 = the contiguous split instead);
        pdl: programmatic dependent launch of the kernel (None = library default, on)."""
        _check(lib().lb_set_option(self._ctx, 3, int(enable)))
        _check(lib().lb_set_option(self._ctx, 4, int(grid)))
        _check(lib().lb_set_option(self._ctx, 5, int(l2_prefetch)))
        _check(lib().lb_set_option(self._ctx, 6, int(wall_weight16)))
        if l2_promotion is not None:
            _check(lib().lb_set_option(self._ctx, 7, int(l2_promotion)))
        _check(lib().lb_set_option(self._ctx, 9, int(tail_weight16)))
        if pdl is not None:
            _check(lib().lb_set_option(self._ctx, 10, int(bool(pdl))))

    def edge_pull(self, in_kernel: bool = True):
        """N > 1 two-step exchange: inside the kernel (edge CTAs wait and stage,
        the default) or a separate k_tb_pull launch first (LB_OPT_TB_EDGE_PULL)."""
        _check(lib().lb_set_option(self._ctx, 8, int(bool(in_kernel))))

    def monitor(self, enable: bool = True):
        """Fused monitors: invariants reduced inside the step kernel (lb_monitor)."""
        _check(lib().lb_monitor(self._ctx, int(enable)))

    def launch_count(self) -> int:
        return int(lib().lb_launch_count(self._ctx))
