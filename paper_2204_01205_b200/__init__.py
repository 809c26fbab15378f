"""B200-native hot path of the model-parallel FNO of arXiv 2204.01205.

Thin Python binding of libfno (include/fno.h).  Argument marshalling only:
every step of the spectral layer runs in the library's sm_100a kernels and
NCCL exchanges.  PyTorch supplies device memory, streams and the process
group used to broadcast the NCCL unique id.  There is no CPU fallback: if
libfno.so is missing or a call fails, an exception is raised.

Functions keep the ABI names without the ``fno_`` prefix:
    Problem, Comm, Plan,
    spectral_conv_fwd, spectral_conv_bwd, layer_fwd, layer_bwd, repartition
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FNO_LIB") or os.path.join(_PKG, "lib", "libfno.so")   # FNO_LIB: A/B builds

FNO_ACT_GELU = 0
FNO_ACT_NONE = 1

_STATUS = {0: "FNO_OK", 1: "FNO_ERR_INVALID_ARGUMENT", 2: "FNO_ERR_PLAN", 3: "FNO_ERR_INVALID_STATE",
           4: "FNO_ERR_CUDA", 5: "FNO_ERR_NCCL", 6: "FNO_ERR_WORKSPACE"}


class FnoError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Problem(ctypes.Structure):
    _fields_ = [("grid", ctypes.c_int64 * 4), ("batch", ctypes.c_int32), ("width", ctypes.c_int32),
                ("modes", ctypes.c_int32 * 4), ("pgrid", ctypes.c_int32 * 2), ("flags", ctypes.c_uint32)]


NET_MAXK = 16


class _NetDesc(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("in_channels", ctypes.c_int32), ("proj_bias", ctypes.c_int32)]


class _NetParams(ctypes.Structure):
    _fields_ = [("Wt", ctypes.c_void_p), ("bt", ctypes.c_void_p), ("Wc", ctypes.c_void_p), ("bc", ctypes.c_void_p),
                ("R", ctypes.c_void_p * NET_MAXK), ("W", ctypes.c_void_p * NET_MAXK), ("b", ctypes.c_void_p * NET_MAXK),
                ("Wp", ctypes.c_void_p), ("bp", ctypes.c_void_p)]


class _NetActs(ctypes.Structure):
    _fields_ = [("nu", ctypes.c_void_p * (NET_MAXK + 1)), ("z", ctypes.c_void_p * NET_MAXK),
                ("vhat", ctypes.c_void_p * NET_MAXK)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libfno.so (built by paper_2204_01205_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} not found: run `python -m paper_2204_01205_b200.build` "
                                    "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
        P = ctypes.POINTER
        sig = {
            "fno_comm_unique_id": [ctypes.c_char_p],
            "fno_comm_init": [ctypes.c_char_p, i32, i32, P(vp)],
            "fno_comm_init_local": [i32, i32, P(vp)],
            "fno_comm_destroy": [vp],
            "fno_comm_size": [vp, P(i32), P(i32)],
            "fno_plan_create": [P(_Problem), vp, P(vp)],
            "fno_plan_destroy": [vp],
            "fno_plan_workspace_size": [vp, P(sz)],
            "fno_plan_set_workspace": [vp, vp, sz],
            "fno_plan_connect_peers": [vp, vp],
            "fno_plan_peer_enabled": [vp, P(i32)],
            "fno_plan_pass_c_info": [vp, i32, P(ctypes.c_int64)],
            "fno_plan_set_pass_c": [vp, i32, i32],
            "fno_plan_local_box": [vp, P(ctypes.c_int64), P(ctypes.c_int64)],
            "fno_plan_set_io_partition": [vp, P(ctypes.c_int32)],
            "fno_plan_io_box": [vp, P(ctypes.c_int64), P(ctypes.c_int64)],
            "fno_plan_owned_modes": [vp, P(ctypes.c_int32), P(ctypes.c_int32)],
            "fno_plan_vhat_elems": [vp, P(sz)],
            "fno_spectral_conv_fwd": [vp, vp, vp, vp, vp, vp],
            "fno_spectral_conv_bwd": [vp, vp, vp, vp, vp, vp, i32, vp],
            "fno_layer_fwd": [vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "fno_layer_bwd": [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp],
            "fno_repartition": [vp, i32, P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_int32), sz, vp, vp, vp,
                                P(sz), vp],
            "fno_net_workspace_size": [vp, P(_NetDesc), P(sz)],
            "fno_net_fwd": [vp, P(_NetDesc), P(_NetParams), vp, P(_NetActs), vp, vp],
            "fno_net_loss": [vp, vp, vp, vp, vp, vp],
            "fno_net_bwd": [vp, P(_NetDesc), P(_NetParams), vp, P(_NetActs), vp, vp, P(_NetParams), vp, vp, vp, vp],
            "fno_comm_allreduce": [vp, vp, sz, i32, vp],
            "fno_group_connect": [i32, vp],
            "fno_group_spectral_conv_fwd": [i32, vp, vp, vp, vp, vp, vp],
            "fno_group_spectral_conv_bwd": [i32, vp, vp, vp, vp, vp, vp, i32, vp],
            "fno_group_layer_fwd": [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp],
            "fno_group_layer_bwd": [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i32, vp],
            "fno_adam": [vp, vp, vp, vp, sz, ctypes.c_float, ctypes.c_float, ctypes.c_float, ctypes.c_float, i32, vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        L.fno_plan_profile_enable.argtypes = [vp, i32]
        L.fno_plan_profile_enable.restype = ctypes.c_int
        L.fno_plan_profile_read.argtypes = [vp, P(ctypes.c_double), P(ctypes.c_int64), i32]
        L.fno_plan_profile_read.restype = ctypes.c_int
        L.fno_profile_stage_count.restype = ctypes.c_int
        L.fno_profile_stage_name.argtypes = [ctypes.c_int]
        L.fno_profile_stage_name.restype = ctypes.c_char_p
        L.fno_kernel_launches.restype = ctypes.c_ulonglong
        L.fno_status_string.argtypes = [ctypes.c_int]
        L.fno_status_string.restype = ctypes.c_char_p
        L.fno_last_error.argtypes = []
        L.fno_last_error.restype = ctypes.c_char_p
        L.fno_abi_version.restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int, where: str):
    if status != 0:
        raise FnoError(status, where, lib().fno_last_error().decode(errors="replace"))


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return t.data_ptr()


def _stream(stream) -> Optional[int]:
    import torch
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


@dataclass
class Problem:
    """Problem statement (P:52 modes per dimension, P:182 grid, P:183 width, P:61 partition)."""
    grid: Sequence[int]                 # global X, Y, Z, T
    width: int                          # C
    modes: Sequence[int]                # mx, my, mz, mt
    batch: int = 1
    pgrid: Sequence[int] = (1, 1)       # px, py
    act: str = "gelu"                   # "gelu" | "none"

    def to_c(self) -> _Problem:
        p = _Problem()
        for i in range(4):
            p.grid[i] = int(self.grid[i])
            p.modes[i] = int(self.modes[i])
        p.batch = int(self.batch)
        p.width = int(self.width)
        p.pgrid[0], p.pgrid[1] = int(self.pgrid[0]), int(self.pgrid[1])
        p.flags = FNO_ACT_NONE if self.act == "none" else FNO_ACT_GELU
        return p


class Comm:
    """NCCL communicator of libfno (one process per GPU)."""

    def __init__(self, handle: int, nranks: int, rank: int):
        self.handle = ctypes.c_void_p(handle)
        self.nranks, self.rank = nranks, rank

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().fno_comm_unique_id(buf), "fno_comm_unique_id")
        return buf.raw

    @classmethod
    def init(cls, uid: bytes, nranks: int, rank: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(lib().fno_comm_init(uid, nranks, rank, ctypes.byref(h)), "fno_comm_init")
        return cls(h.value, nranks, rank)

    @classmethod
    def local(cls, nranks: int, rank: int) -> "Comm":
        h = ctypes.c_void_p()
        _check(lib().fno_comm_init_local(nranks, rank, ctypes.byref(h)), "fno_comm_init_local")
        return cls(h.value, nranks, rank)

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Create on every rank of a torch.distributed group (id broadcast from rank 0)."""
        import torch
        import torch.distributed as dist
        rank, n = dist.get_rank(group), dist.get_world_size(group)
        uid = cls.unique_id() if rank == 0 else bytes(128)
        dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else "cpu"
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        return cls.init(bytes(t.cpu().tolist()), n, rank)

    def destroy(self):
        if self.handle:
            lib().fno_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Plan:
    """fno_plan_t plus its caller-owned workspace (a torch uint8 tensor)."""

    def __init__(self, problem: Problem, comm: Optional[Comm] = None, device=None, allocate: bool = True,
                 peer_exchange: Optional[bool] = None, io_pgrid: Optional[Sequence[int]] = None):
        """io_pgrid: optional caller-side (px, py, pz, pt) partition of the fields
        (fno_plan_set_io_partition, App. A 3-D / temporal partitions)."""
        self.problem = problem
        self.comm = comm
        h = ctypes.c_void_p()
        c = problem.to_c()
        _check(lib().fno_plan_create(ctypes.byref(c), comm.handle if comm else None, ctypes.byref(h)), "fno_plan_create")
        self.handle = h
        self.io_pgrid = None
        if io_pgrid is not None:
            arr = (ctypes.c_int32 * 4)(*[int(x) for x in io_pgrid])
            _check(lib().fno_plan_set_io_partition(h, arr), "fno_plan_set_io_partition")
            self.io_pgrid = tuple(int(x) for x in io_pgrid)
        self.workspace = None
        if allocate:
            import torch
            dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
            self.workspace = torch.empty(max(self.workspace_size(), 256), dtype=torch.uint8, device=dev)
            _check(lib().fno_plan_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
                   "fno_plan_set_workspace")
            # direct NVLink stores for the pencil repartitions (collective; FNO_PEER_EXCHANGE=0 keeps
            # the NCCL send/recv exchanges)
            if peer_exchange is None:
                peer_exchange = os.environ.get("FNO_PEER_EXCHANGE", "1") != "0"
            if comm is not None and peer_exchange and self._nranks() > 1:
                self.connect_peers()

    def _nranks(self) -> int:
        n, r = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().fno_comm_size(self.comm.handle, ctypes.byref(n), ctypes.byref(r)), "fno_comm_size")
        return n.value

    def connect_peers(self):
        """Collective: map the peers' workspaces (fno_plan_connect_peers)."""
        import torch
        _check(lib().fno_plan_connect_peers(self.handle, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "fno_plan_connect_peers")

    def peer_enabled(self) -> bool:
        """True if the exchanges are direct NVLink peer stores (collective decision)."""
        e = ctypes.c_int32()
        _check(lib().fno_plan_peer_enabled(self.handle, ctypes.byref(e)), "fno_plan_peer_enabled")
        return bool(e.value)

    def workspace_size(self) -> int:
        n = ctypes.c_size_t()
        _check(lib().fno_plan_workspace_size(self.handle, ctypes.byref(n)), "fno_plan_workspace_size")
        return n.value

    def local_box(self):
        lo = (ctypes.c_int64 * 4)()
        hi = (ctypes.c_int64 * 4)()
        _check(lib().fno_plan_local_box(self.handle, lo, hi), "fno_plan_local_box")
        return list(zip(lo, hi))

    def io_box(self):
        """This rank's box of the io partition (== local_box without one)."""
        lo = (ctypes.c_int64 * 4)()
        hi = (ctypes.c_int64 * 4)()
        _check(lib().fno_plan_io_box(self.handle, lo, hi), "fno_plan_io_box")
        return list(zip(lo, hi))

    def io_shape(self):
        box = self.io_box() if self.io_pgrid is not None else self.local_box()
        return (self.problem.batch, self.problem.width) + tuple(hi - lo for lo, hi in box)

    def owned_modes(self):
        a, b = ctypes.c_int32(), ctypes.c_int32()
        _check(lib().fno_plan_owned_modes(self.handle, ctypes.byref(a), ctypes.byref(b)), "fno_plan_owned_modes")
        return a.value, b.value

    def vhat_elems(self) -> int:
        n = ctypes.c_size_t()
        _check(lib().fno_plan_vhat_elems(self.handle, ctypes.byref(n)), "fno_plan_vhat_elems")
        return n.value

    def local_shape(self):
        box = self.local_box()
        return (self.problem.batch, self.problem.width) + tuple(hi - lo for lo, hi in box)

    def weight_shape(self):
        lo, hi = self.owned_modes()
        mx, my, mz, mt = self.problem.modes
        C = self.problem.width
        return (C, C, 2 * mx, 2 * my, hi - lo, mt)

    def vhat_shape(self):
        s = self.weight_shape()
        return (self.problem.batch,) + s[1:]

    def profile_enable(self, on: bool = True):
        _check(lib().fno_plan_profile_enable(self.handle, int(bool(on))), "fno_plan_profile_enable")

    def profile_read(self):
        """{stage name: (total ms, launches)} since the last read (waits for the events)."""
        n = lib().fno_profile_stage_count()
        ms = (ctypes.c_double * n)()
        cnt = (ctypes.c_int64 * n)()
        _check(lib().fno_plan_profile_read(self.handle, ms, cnt, n), "fno_plan_profile_read")
        return {lib().fno_profile_stage_name(i).decode(): (ms[i], cnt[i]) for i in range(n) if cnt[i]}

    def destroy(self):
        if self.handle:
            lib().fno_plan_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def plan_pass_c_kernels(plan: Plan) -> dict:
    """{mode: {family, width, stages, smem}} of the pass C kernels the plan selected."""
    fam = {5: "split (dv: the forward kernel with W^T; dW, db: dw_partial)",
           4: "pass_c4 (warp-specialised, TMA ring, tcgen05)", 3: "pass_c3 (tcgen05 1x1)", 2: "pass_c2 (FFMA)",
           1: "pass_c (generic)"}
    out = {}
    for m, name in enumerate(("u", "fwd", "bwd")):
        info = (ctypes.c_int64 * 4)()
        _check(lib().fno_plan_pass_c_info(plan.handle, m, info), "fno_plan_pass_c_info")
        out[name] = {"family": fam.get(info[0], info[0]), "width": info[1], "stages": info[2] & 255,
                     "smem": info[3]}
        if info[0] == 5:   # the configuration of its dv kernel (the forward family's)
            out[name]["dv_kernel"] = out["fwd"]["family"]
        if info[0] in (4, 5) and info[2] >> 8:
            out[name]["u_buffers"] = (info[2] >> 8) & 255
            out[name]["slab_staged"] = bool((info[2] >> 16) & 1)
    return out


def plan_set_pass_c(plan: Plan, mode: str, family: int):
    """Force the pass C kernel family (1 pass_c, 2 pass_c2, 3 pass_c3, 4 pass_c4; 5 the split backward:
    dv by the forward family's kernel with W^T, dW / db by dw_partial) for mode "u" / "fwd" / "bwd"
    (A/B runs and tests; the plan's default is the measured-fastest eligible family)."""
    m = {"u": 0, "fwd": 1, "bwd": 2}[mode]
    _check(lib().fno_plan_set_pass_c(plan.handle, m, int(family)), "fno_plan_set_pass_c")


def kernel_launches() -> int:
    """Kernels launched through libfno by this process so far."""
    return int(lib().fno_kernel_launches())


def _contig(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ValueError("libfno expects contiguous tensors")


def spectral_conv_fwd(plan: Plan, v, R, u, vhat_save=None, stream=None):
    """u = S v (Eq. 3 / P:121 Eq. sconv_dist)."""
    _contig(v, R, u, vhat_save)
    _check(lib().fno_spectral_conv_fwd(plan.handle, _ptr(v), _ptr(R), _ptr(u), _ptr(vhat_save), _stream(stream)),
           "fno_spectral_conv_fwd")


def spectral_conv_bwd(plan: Plan, g, R, vhat_saved=None, dv=None, dR=None, accumulate=False, stream=None):
    """dv = S^T g and dR (+)= (c/N) sum_b conj(V^) G^."""
    _contig(g, R, vhat_saved, dv, dR)
    _check(lib().fno_spectral_conv_bwd(plan.handle, _ptr(g), _ptr(R), _ptr(vhat_saved), _ptr(dv), _ptr(dR),
                                       int(bool(accumulate)), _stream(stream)), "fno_spectral_conv_bwd")


def layer_fwd(plan: Plan, v, R, W, b, y, z_save=None, vhat_save=None, stream=None):
    """y = sigma(W v + b + S v) (Eq. dist_block)."""
    _contig(v, R, W, b, y, z_save, vhat_save)
    _check(lib().fno_layer_fwd(plan.handle, _ptr(v), _ptr(R), _ptr(W), _ptr(b), _ptr(y), _ptr(z_save),
                               _ptr(vhat_save), _stream(stream)), "fno_layer_fwd")


def layer_bwd(plan: Plan, v, z_saved, vhat_saved, dy, R, W, dv, dR, dW, db=None, accumulate=False, stream=None):
    """Backward of the DFNO block; dW, db summed over all ranks."""
    _contig(v, z_saved, vhat_saved, dy, R, W, dv, dR, dW, db)
    _check(lib().fno_layer_bwd(plan.handle, _ptr(v), _ptr(z_saved), _ptr(vhat_saved), _ptr(dy), _ptr(R), _ptr(W),
                               _ptr(dv), _ptr(dR), _ptr(dW), _ptr(db), int(bool(accumulate)), _stream(stream)),
           "fno_layer_bwd")


# ---- whole network (fno_net_*) --------------------------------

def _net_desc(layers: int, in_channels: int, proj_bias: bool) -> _NetDesc:
    return _NetDesc(int(layers), int(in_channels), int(bool(proj_bias)))


def _net_params(P: dict) -> _NetParams:
    """P: Wt [T], bt [T], Wc [C, Cin], bc [C], R/W/b lists, Wp [C], bp [1] or None."""
    c = _NetParams()
    c.Wt, c.bt, c.Wc, c.bc = _ptr(P["Wt"]), _ptr(P["bt"]), _ptr(P["Wc"]), _ptr(P["bc"])
    for k in range(len(P["R"])):
        c.R[k], c.W[k], c.b[k] = _ptr(P["R"][k]), _ptr(P["W"][k]), _ptr(P["b"][k])
    c.Wp, c.bp = _ptr(P["Wp"]), _ptr(P.get("bp"))
    return c


def _net_acts(A: dict) -> _NetActs:
    c = _NetActs()
    for k, t in enumerate(A["nu"]):
        c.nu[k] = _ptr(t)
    for k, t in enumerate(A["z"]):
        c.z[k] = _ptr(t)
    for k, t in enumerate(A["vhat"]):
        c.vhat[k] = _ptr(t)
    return c


def net_workspace_size(plan: Plan, layers: int, in_channels: int, proj_bias: bool = True) -> int:
    d = _net_desc(layers, in_channels, proj_bias)
    n = ctypes.c_size_t()
    _check(lib().fno_net_workspace_size(plan.handle, ctypes.byref(d), ctypes.byref(n)), "fno_net_workspace_size")
    return n.value


def net_fwd(plan: Plan, params: dict, a, acts: dict, u, in_channels: int, proj_bias: bool = True, stream=None):
    """Lift, K blocks, projection."""
    d = _net_desc(len(params["R"]), in_channels, proj_bias)
    cp, ca = _net_params(params), _net_acts(acts)
    _check(lib().fno_net_fwd(plan.handle, ctypes.byref(d), ctypes.byref(cp), _ptr(a), ctypes.byref(ca), _ptr(u),
                             _stream(stream)), "fno_net_fwd")


def net_loss(plan: Plan, u, y, loss3, net_ws, stream=None):
    """loss3 = {||u - y|| / ||y||, ||u - y||^2, ||y||^2} over all ranks."""
    _check(lib().fno_net_loss(plan.handle, _ptr(u), _ptr(y), _ptr(loss3), _ptr(net_ws), _stream(stream)),
           "fno_net_loss")


def net_bwd(plan: Plan, params: dict, a, acts: dict, u, y, grads: dict, scratch0, scratch1, net_ws, in_channels: int,
            proj_bias: bool = True, stream=None):
    """Gradient of the loss w.r.t. every parameter (after net_loss on the same u, y, net_ws)."""
    d = _net_desc(len(params["R"]), in_channels, proj_bias)
    cp, ca, cg = _net_params(params), _net_acts(acts), _net_params(grads)
    _check(lib().fno_net_bwd(plan.handle, ctypes.byref(d), ctypes.byref(cp), _ptr(a), ctypes.byref(ca), _ptr(u),
                             _ptr(y), ctypes.byref(cg), _ptr(scratch0), _ptr(scratch1), _ptr(net_ws), _stream(stream)),
           "fno_net_bwd")


def comm_allreduce(comm: Comm, t, average: bool = True, stream=None):
    """In-place NCCL all-reduce (mean or sum) of a float32 / complex64 tensor over comm
    (data-parallel gradient averaging across replicas)."""
    n = t.numel() * (2 if t.is_complex() else 1)
    _check(lib().fno_comm_allreduce(comm.handle, _ptr(t), n, int(bool(average)), _stream(stream)),
           "fno_comm_allreduce")


def adam(p, g, m, v, step: int, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
    """One Adam step on a float32 (or complex64, as 2n floats) tensor."""
    n = p.numel() * (2 if p.is_complex() else 1)
    _check(lib().fno_adam(_ptr(p), _ptr(g), _ptr(m), _ptr(v), n, lr, beta1, beta2, eps, int(step), _stream(stream)),
           "fno_adam")


# ---- plan groups: a P-rank decomposition in one process on one device ---------

def _parr(ts):
    """ctypes array of device pointers (None -> NULL entry); None -> NULL array."""
    if ts is None:
        return None
    return (ctypes.c_void_p * len(ts))(*[_ptr(t) for t in ts])


class PlanGroup:
    """The P ranks of an x/y decomposition (pgrid (px, py)) as P plans on one
    device (fno_group_connect).  ``plans[r]`` gives rank r's local box, owned kz
    block and shapes; the compute calls take one tensor per rank."""

    def __init__(self, problem: Problem, device=None):
        n = int(problem.pgrid[0]) * int(problem.pgrid[1])
        self.problem, self.n = problem, n
        self.comms = [Comm.local(n, r) for r in range(n)]
        self.plans = [Plan(problem, self.comms[r], device=device, peer_exchange=False) for r in range(n)]
        self._h = (ctypes.c_void_p * n)(*[p.handle.value for p in self.plans])
        _check(lib().fno_group_connect(n, self._h), "fno_group_connect")

    def destroy(self):
        for p in self.plans:
            p.destroy()
        for c in self.comms:
            c.destroy()


def group_spectral_conv_fwd(g: PlanGroup, vs, Rs, us, vhs=None, stream=None):
    _check(lib().fno_group_spectral_conv_fwd(g.n, g._h, _parr(vs), _parr(Rs), _parr(us), _parr(vhs), _stream(stream)),
           "fno_group_spectral_conv_fwd")


def group_spectral_conv_bwd(g: PlanGroup, gs, Rs, vhs=None, dvs=None, dRs=None, accumulate=False, stream=None):
    _check(lib().fno_group_spectral_conv_bwd(g.n, g._h, _parr(gs), _parr(Rs), _parr(vhs), _parr(dvs), _parr(dRs),
                                             int(bool(accumulate)), _stream(stream)), "fno_group_spectral_conv_bwd")


def group_layer_fwd(g: PlanGroup, vs, Rs, W, b, ys, zs=None, vhs=None, stream=None):
    _check(lib().fno_group_layer_fwd(g.n, g._h, _parr(vs), _parr(Rs), _ptr(W), _ptr(b), _parr(ys), _parr(zs),
                                     _parr(vhs), _stream(stream)), "fno_group_layer_fwd")


def group_layer_bwd(g: PlanGroup, vs, zs, vhs, dys, Rs, W, dvs, dRs, dW, db=None, accumulate=False, stream=None):
    _check(lib().fno_group_layer_bwd(g.n, g._h, _parr(vs), _parr(zs), _parr(vhs), _parr(dys), _parr(Rs), _ptr(W),
                                     _parr(dvs), _parr(dRs), _ptr(dW), _ptr(db), int(bool(accumulate)),
                                     _stream(stream)), "fno_group_layer_bwd")


def repartition(comm: Optional[Comm], global_shape, src_pgrid, dst_pgrid, src_local, dst_local, stream=None):
    """R_{P->Q}; the adjoint is the call with the pgrids swapped."""
    import torch
    nd = len(global_shape)
    shp = (ctypes.c_int64 * nd)(*[int(s) for s in global_shape])
    sp = (ctypes.c_int32 * nd)(*[int(s) for s in src_pgrid])
    dp = (ctypes.c_int32 * nd)(*[int(s) for s in dst_pgrid])
    eb = src_local.element_size()
    n = ctypes.c_size_t(0)
    h = comm.handle if comm else None
    _check(lib().fno_repartition(h, nd, shp, sp, dp, eb, None, None, None, ctypes.byref(n), None),
           "fno_repartition(size)")
    ws = torch.empty(max(n.value, 256), dtype=torch.uint8, device=src_local.device)
    n2 = ctypes.c_size_t(ws.numel())
    _contig(src_local, dst_local)
    _check(lib().fno_repartition(h, nd, shp, sp, dp, eb, _ptr(src_local), _ptr(dst_local), ws.data_ptr(),
                                 ctypes.byref(n2), _stream(stream)), "fno_repartition")
    return ws  # keep alive until the stream has consumed it


__all__ = ["Problem", "Comm", "Plan", "PlanGroup", "FnoError", "lib", "spectral_conv_fwd", "spectral_conv_bwd",
           "layer_fwd", "layer_bwd", "group_spectral_conv_fwd", "group_spectral_conv_bwd", "group_layer_fwd",
           "group_layer_bwd", "repartition", "kernel_launches", "LIB_PATH"]
