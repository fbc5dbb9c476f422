"""Thin ctypes binding of libpic (include/pic.h).  Argument marshalling only:
every step of the particle path runs in the CUDA kernels of libpic.so.

The functions keep the C names (pic_init, pic_mover, pic_moments, pic_exchange,
...).  `Context` is a convenience owner of one pic_ctx plus its torch-allocated
device workspace.  PyTorch supplies device memory, the stream and (for
multi-GPU) the process group that broadcasts the NCCL id; nothing else.

If libpic.so is missing or no CUDA device is present this module raises: there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional, Sequence

import torch

from . import inputs as _inputs  # noqa: F401  (re-export convenience for callers)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIC_LIB", os.path.join(HERE, "libpic.so"))

PIC_MAX_SPECIES = 8
PIC_NCCL_ID_BYTES = 128
PIC_OK, PIC_EINVAL, PIC_ECUDA, PIC_ENCCL, PIC_ENOMEM, PIC_ESTATE, PIC_ERANGE, PIC_ENONFINITE = range(8)
STATUS_NAMES = ["PIC_OK", "PIC_EINVAL", "PIC_ECUDA", "PIC_ENCCL", "PIC_ENOMEM", "PIC_ESTATE",
                "PIC_ERANGE", "PIC_ENONFINITE"]
KERNEL_AUTO, KERNEL_BASIC, KERNEL_TILED = 0, 1, 2
TRANSPORT_AUTO, TRANSPORT_NCCL, TRANSPORT_PEER, TRANSPORT_LOOPBACK = 0, 1, 2, 3
STAT_NAMES = ["removed", "sent", "received", "far", "clamped", "nonfinite", "overflow", "multiwrap"]
EXPORTS = ["pic_abi_version", "pic_nccl_id", "pic_workspace_bytes", "pic_init", "pic_loopback_link", "pic_set_stream",
           "pic_set_particles", "pic_add_particles", "pic_count", "pic_get_particles", "pic_set_fields", "pic_mover",
           "pic_moments", "pic_exchange", "pic_cycle", "pic_set_graph", "pic_moment_shape", "pic_get_moments",
           "pic_sync", "pic_get_moments_async", "pic_join_copies", "pic_implicit_sources", "pic_set_injection", "pic_control", "pic_gmm", "pic_moment_ptr", "pic_get_transport", "pic_launch_count", "pic_profile", "pic_profile_read", "pic_last_error", "pic_destroy"]


class pic_config(C.Structure):
    _fields_ = [
        ("ncell", C.c_int64 * 3), ("len", C.c_double * 3), ("bc", C.c_int32 * 3),
        ("dt", C.c_double), ("c", C.c_double), ("n_species", C.c_int32),
        ("qom", C.c_double * PIC_MAX_SPECIES), ("n_iter", C.c_int32 * PIC_MAX_SPECIES),
        ("capacity", C.c_int64 * PIC_MAX_SPECIES),
        ("planet_center", C.c_double * 3), ("planet_radius", C.c_double),
        ("rank", C.c_int32), ("nranks", C.c_int32), ("slab_lo", C.c_int64), ("slab_hi", C.c_int64),
        ("ghost", C.c_int32), ("transport", C.c_int32), ("kernel", C.c_int32), ("relativistic", C.c_int32),
        ("far_hops", C.c_int32), ("barrier_timeout_ms", C.c_int32),
    ]


class PicError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 8 else status}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libpic.so; raise if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise ImportError(f"libpic.so not built at {path}: run __graft_entry__.build()")
        lib = C.CDLL(path)
        P = C.POINTER
        vp = C.c_void_p
        lib.pic_abi_version.restype = C.c_int32
        lib.pic_nccl_id.argtypes = [vp]
        lib.pic_workspace_bytes.argtypes = [P(pic_config), P(C.c_int64)]
        lib.pic_init.argtypes = [P(pic_config), vp, vp, C.c_int64, P(vp)]
        lib.pic_set_stream.argtypes = [vp, vp]
        lib.pic_loopback_link.argtypes = [P(vp), C.c_int32]
        lib.pic_set_particles.argtypes = [vp, C.c_int32, C.c_int64, P(vp), vp]
        lib.pic_add_particles.argtypes = [vp, C.c_int32, C.c_int64, P(vp), vp]
        lib.pic_count.argtypes = [vp, C.c_int32, P(C.c_int64)]
        lib.pic_get_particles.argtypes = [vp, C.c_int32, P(vp), vp]
        lib.pic_set_fields.argtypes = [vp, vp]
        lib.pic_mover.argtypes = [vp, C.c_int32]
        lib.pic_moments.argtypes = [vp, C.c_int32]
        lib.pic_exchange.argtypes = [vp]
        lib.pic_cycle.argtypes = [vp]
        lib.pic_set_graph.argtypes = [vp, C.c_int32]
        lib.pic_moment_shape.argtypes = [vp, P(C.c_int64)]
        lib.pic_get_moments.argtypes = [vp, C.c_int32, vp]
        lib.pic_sync.argtypes = [vp, P(C.c_int64)]
        lib.pic_launch_count.argtypes = [vp, P(C.c_int64)]
        lib.pic_get_transport.argtypes = [vp, P(C.c_int32)]
        lib.pic_get_moments_async.argtypes = [vp, C.c_int32, vp]
        lib.pic_join_copies.argtypes = [vp]
        lib.pic_implicit_sources.argtypes = [vp, vp, vp, vp]
        lib.pic_set_injection.argtypes = [vp, C.c_int32, C.c_int32, C.c_double, P(C.c_double), C.c_double,
                                          C.c_uint64]
        lib.pic_control.argtypes = [vp, C.c_int32, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                    P(C.c_int32)]
        lib.pic_gmm.argtypes = [vp, C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32, vp, vp, vp, vp,
                                P(C.c_int64)]
        lib.pic_moment_ptr.argtypes = [vp, C.c_int32, C.c_int32, P(vp), P(C.c_int64), P(C.c_int64),
                                       P(C.c_double)]
        lib.pic_profile.argtypes = [vp, C.c_int32]
        lib.pic_profile_read.argtypes = [vp, P(C.c_double), P(C.c_int64)]
        lib.pic_last_error.argtypes = [vp]
        lib.pic_last_error.restype = C.c_char_p
        lib.pic_destroy.argtypes = [vp]
        for name in EXPORTS:
            if name not in ("pic_abi_version", "pic_last_error"):
                getattr(lib, name).restype = C.c_int
        _lib = lib
    return _lib


def _check(st, ctx=None, what=""):
    if st != PIC_OK:
        msg = what
        if ctx:
            msg += ": " + load_library().pic_last_error(ctx).decode()
        raise PicError(st, msg)


# ------------------------------------------------------------ C-name layer --
def pic_nccl_id() -> bytes:
    buf = (C.c_uint8 * PIC_NCCL_ID_BYTES)()
    _check(load_library().pic_nccl_id(C.cast(buf, C.c_void_p)), what="pic_nccl_id")
    return bytes(buf)


def pic_workspace_bytes(cfg: pic_config) -> int:
    out = C.c_int64()
    _check(load_library().pic_workspace_bytes(C.byref(cfg), C.byref(out)), what="pic_workspace_bytes")
    return out.value


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def make_config(w, *, rank=0, nranks=1, capacity=None, ghost=2, transport=TRANSPORT_AUTO, kernel=KERNEL_AUTO,
                n_iter=None, relativistic=None, far_hops=0, barrier_timeout_ms=0) -> pic_config:
    """pic_config from an inputs.Workload (marshalling only)."""
    cfg = pic_config()
    lo, hi = w.slab_or_all()
    for d in range(3):
        cfg.ncell[d] = w.ncell[d]
        cfg.len[d] = w.length[d]
        cfg.bc[d] = w.bc[d]
        cfg.planet_center[d] = w.planet_center[d]
    cfg.dt, cfg.c, cfg.planet_radius = w.dt, w.c, w.planet_radius
    cfg.n_species = len(w.species)
    for s, sp in enumerate(w.species):
        cfg.qom[s] = sp.qom
        cfg.n_iter[s] = n_iter if n_iter is not None else w.n_iter
        cfg.capacity[s] = capacity[s] if capacity is not None else 0
    cfg.rank, cfg.nranks, cfg.slab_lo, cfg.slab_hi = rank, nranks, lo, hi
    cfg.ghost, cfg.transport, cfg.kernel = ghost, transport, kernel
    cfg.relativistic = int(bool(getattr(w, "relativistic", False) if relativistic is None else relativistic))
    cfg.far_hops = int(far_hops)
    cfg.barrier_timeout_ms = int(barrier_timeout_ms)
    return cfg


def pic_loopback_link(contexts: Sequence["Context"]):
    """Join the slab contexts of a loopback decomposition (TRANSPORT_LOOPBACK,
    contexts[r] = rank r, one device).  Each context must keep its own stream
    and be stepped from its own host thread (the flag barriers spin on the
    device, as between ranks)."""
    arr = (C.c_void_p * len(contexts))(*[c.h.value for c in contexts])
    _check(load_library().pic_loopback_link(arr, len(contexts)), contexts[0].h, "pic_loopback_link")


class Context:
    """One pic_ctx + its workspace tensor on the current CUDA device."""

    def __init__(self, cfg: pic_config, nccl_id: Optional[bytes] = None, stream=None):
        if not torch.cuda.is_available():
            raise RuntimeError("libpic needs a CUDA device (there is no CPU path)")
        self.lib = load_library()
        self.cfg = cfg
        nbytes = pic_workspace_bytes(cfg)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_uint8 * PIC_NCCL_ID_BYTES).from_buffer_copy(nccl_id)
        st = self.lib.pic_init(C.byref(cfg), C.cast(idbuf, C.c_void_p) if idbuf is not None else None,
                               C.c_void_p(self.workspace.data_ptr()), nbytes, C.byref(h))
        _check(st, what="pic_init")
        self.h = h
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        _check(self.lib.pic_set_stream(self.h, C.c_void_p(self.stream.cuda_stream)), self.h, "pic_set_stream")

    # -- particles
    def set_particles(self, s: int, parts: Dict[str, torch.Tensor]):
        arrs = [parts[k] for k in "xyzuvwq"]
        n = arrs[0].numel()
        for a in arrs:
            assert a.dtype == torch.float64 and a.is_contiguous() and a.numel() == n
        P7 = (C.c_void_p * 7)(*[a.data_ptr() for a in arrs])
        idt = parts.get("id")
        if idt is not None:
            assert idt.dtype == torch.int64 and idt.is_contiguous() and idt.numel() == n
        _check(self.lib.pic_set_particles(self.h, s, n, P7, _ptr(idt)), self.h, "pic_set_particles")

    def add_particles(self, s: int, parts: Dict[str, torch.Tensor]):
        """Append particles to species s (pic_add_particles)."""
        arrs = [parts[k] for k in "xyzuvwq"]
        n = arrs[0].numel()
        for a in arrs:
            assert a.dtype == torch.float64 and a.is_contiguous() and a.numel() == n
        P7 = (C.c_void_p * 7)(*[a.data_ptr() for a in arrs])
        idt = parts.get("id")
        if idt is not None:
            assert idt.dtype == torch.int64 and idt.is_contiguous() and idt.numel() == n
        _check(self.lib.pic_add_particles(self.h, s, n, P7, _ptr(idt)), self.h, "pic_add_particles")

    def count(self, s: int) -> int:
        out = C.c_int64()
        _check(self.lib.pic_count(self.h, s, C.byref(out)), self.h, "pic_count")
        return out.value

    def get_particles(self, s: int, device="cuda") -> Dict[str, torch.Tensor]:
        n = self.count(s)
        out = {k: torch.empty(n, dtype=torch.float64, device=device) for k in "xyzuvwq"}
        out["id"] = torch.empty(n, dtype=torch.int64, device=device)
        P7 = (C.c_void_p * 7)(*[out[k].data_ptr() for k in "xyzuvwq"])
        _check(self.lib.pic_get_particles(self.h, s, P7, _ptr(out["id"])), self.h, "pic_get_particles")
        return out

    # -- fields / steps
    def set_fields(self, EB: torch.Tensor):
        assert EB.dtype == torch.float64 and EB.is_contiguous()
        _check(self.lib.pic_set_fields(self.h, _ptr(EB)), self.h, "pic_set_fields")

    def mover(self, s: int = -1):
        _check(self.lib.pic_mover(self.h, s), self.h, "pic_mover")

    def moments(self, s: int = -1):
        _check(self.lib.pic_moments(self.h, s), self.h, "pic_moments")

    def exchange(self):
        _check(self.lib.pic_exchange(self.h), self.h, "pic_exchange")

    def cycle(self):
        _check(self.lib.pic_cycle(self.h), self.h, "pic_cycle")

    def set_graph(self, enable: bool = True):
        """pic_set_graph: replay whole cycles from CUDA graphs where possible."""
        _check(self.lib.pic_set_graph(self.h, 1 if enable else 0), self.h, "pic_set_graph")

    def moment_shape(self):
        out = (C.c_int64 * 3)()
        _check(self.lib.pic_moment_shape(self.h, out), self.h, "pic_moment_shape")
        return tuple(out)

    def get_moments(self, s: int, out: Optional[torch.Tensor] = None, device="cuda") -> torch.Tensor:
        nx, ny, nz = self.moment_shape()
        if out is None:
            out = torch.empty((10, nz, ny, nx), dtype=torch.float64, device=device)
        _check(self.lib.pic_get_moments(self.h, s, _ptr(out)), self.h, "pic_get_moments")
        return out

    def get_moments_async(self, s: int, out: torch.Tensor) -> torch.Tensor:
        """Enqueue the copy-out of species s into `out` (pinned host or device);
        complete after join_copies() + a stream synchronisation, or sync()."""
        nx, ny, nz = self.moment_shape()
        assert out.dtype == torch.float64 and out.numel() == 10 * nx * ny * nz and out.is_contiguous()
        _check(self.lib.pic_get_moments_async(self.h, s, _ptr(out)), self.h, "pic_get_moments_async")
        return out

    def implicit_sources(self, device="cuda"):
        """NEXT-2 (Eq. 5-6): (chi[9][nz][ny][nx], rho_hat[nz][ny][nx], J_hat[3][nz][ny][nx])."""
        nx, ny, nz = self.moment_shape()
        chi = torch.empty((9, nz, ny, nx), dtype=torch.float64, device=device)
        rh = torch.empty((nz, ny, nx), dtype=torch.float64, device=device)
        jh = torch.empty((3, nz, ny, nx), dtype=torch.float64, device=device)
        _check(self.lib.pic_implicit_sources(self.h, _ptr(chi), _ptr(rh), _ptr(jh)), self.h, "pic_implicit_sources")
        return chi, rh, jh

    def set_injection(self, s: int, ppc: int, vth: float, drift, q: float, seed: int):
        """NEXT-3 inflow injection of species s at the open x = 0 face."""
        dr = (C.c_double * 3)(*[float(v) for v in drift])
        _check(self.lib.pic_set_injection(self.h, s, int(ppc), float(vth), dr, float(q), int(seed)), self.h,
               "pic_set_injection")

    def control(self, s: int, target: int, theta: float, eps: float, dv: float, seed: int) -> int:
        """NEXT-3 particle control of species s; returns 0 (none), 1 (split), 2 (coalesced)."""
        act = C.c_int32()
        _check(self.lib.pic_control(self.h, s, int(target), float(theta), float(eps), float(dv), int(seed),
                                    C.byref(act)), self.h, "pic_control")
        return act.value

    def gmm(self, s: int, B: int, vmax: float, M: int, n_em: int):
        """NEXT-4: (alpha[M], mu[M][3], sigma[M][6], hist[B][B][B], clipped) as numpy arrays."""
        import numpy as np
        a, mu, sg = np.zeros(M), np.zeros((M, 3)), np.zeros((M, 6))
        h = np.zeros((B, B, B))
        clipped = C.c_int64()
        _check(self.lib.pic_gmm(self.h, s, int(B), float(vmax), int(M), int(n_em), a.ctypes.data, mu.ctypes.data,
                                sg.ctypes.data, h.ctypes.data, C.byref(clipped)), self.h, "pic_gmm")
        return a, mu, sg, h, clipped.value

    def moment_view(self, s: int, comp: int):
        """(view, scale): a zero-copy [nz][ny][nx] view of the RAW sums
        sum q S {1, v, vv} of moment component comp of species s (valid until the
        next moments call) and the R13 normalisation scale = 1/V that turns them
        into the moment (pic_moment_ptr; the binding does no arithmetic on them)."""
        ptr = C.c_void_p()
        st = (C.c_int64 * 3)()
        org = (C.c_int64 * 3)()
        scale = C.c_double()
        _check(self.lib.pic_moment_ptr(self.h, s, comp, C.byref(ptr), st, org, C.byref(scale)), self.h,
               "pic_moment_ptr")
        nx, ny, nz = self.moment_shape()
        base = self.workspace
        off = (ptr.value - base.data_ptr()) // 8
        flat = base[: (base.numel() // 8) * 8].view(torch.float64)
        view = torch.as_strided(flat, (nz, ny, nx), (st[2], st[1], st[0]), off)
        return view, scale.value

    def join_copies(self):
        """The context stream waits (on the device) for all enqueued copies."""
        _check(self.lib.pic_join_copies(self.h), self.h, "pic_join_copies")

    def sync(self, raise_on_error: bool = True) -> Dict[str, int]:
        st_arr = (C.c_int64 * 8)()
        st = self.lib.pic_sync(self.h, st_arr)
        stats = dict(zip(STAT_NAMES, list(st_arr)))
        if raise_on_error:
            _check(st, self.h, f"pic_sync {stats}")
        return stats

    def launch_count(self) -> int:
        out = C.c_int64()
        _check(self.lib.pic_launch_count(self.h, C.byref(out)), self.h, "pic_launch_count")
        return out.value

    @property
    def transport(self) -> int:
        """TRANSPORT_PEER / _NCCL / _LOOPBACK in use (nranks > 1), TRANSPORT_AUTO for one rank."""
        out = C.c_int32()
        _check(self.lib.pic_get_transport(self.h, C.byref(out)), self.h, "pic_get_transport")
        return out.value

    @property
    def peer(self) -> bool:
        return self.transport in (TRANSPORT_PEER, TRANSPORT_LOOPBACK)

    def profile(self, enable: bool = True):
        _check(self.lib.pic_profile(self.h, 1 if enable else 0), self.h, "pic_profile")

    def profile_read(self):
        """{phase: (ms, launches)} for mover, order, deposit, exchange (ghost
        sums + folds), migrate_pre / migrate_post (before / after the count sync)."""
        names = ("mover", "order", "deposit", "exchange", "migrate_pre", "migrate_post", "inject")
        ms = (C.c_double * len(names))()
        n = (C.c_int64 * len(names))()
        _check(self.lib.pic_profile_read(self.h, ms, n), self.h, "pic_profile_read")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def close(self):
        if getattr(self, "h", None):
            self.lib.pic_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
