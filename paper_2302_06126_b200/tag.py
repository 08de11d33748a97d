"""ctypes binding of libtag.so — the C ABI declared in include/tag.h.

Argument marshalling only: tensors are checked (device, dtype, shape, contiguity) and their data
pointers handed to the library; every step of the SFB path runs in libtag's CUDA kernels or in
NCCL. There is no fallback: if libtag.so is missing, importing this module raises; if CUDA is
unavailable, every compute call raises TagError.
"""
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# TAG_LIB_PATH: load an experimental build instead (diagnostics/sweeps only)
LIB_PATH = os.environ.get("TAG_LIB_PATH") or os.path.join(_HERE, "libtag.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libtag.so not built ({LIB_PATH}); run __graft_entry__.build() or "
                      f"`make -C {os.path.join(_HERE, 'csrc')}`")
_lib = ctypes.CDLL(LIB_PATH)

# ------------------------------------------------------------------ enums (tag.h)
OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_NCCL, ERR_OOM, ERR_NOT_INITIALIZED, ERR_ASYNC = \
    range(8)
F32, BF16 = 0, 1
SYNC_ALLREDUCE, SYNC_SFB, SYNC_NONE, SYNC_PS = 0, 1, 2, 3
RULE_NORTHSTAR, RULE_PAPER_ILP, RULE_WIRE = 0, 1, 2

_TORCH_DT = {F32: torch.float32, BF16: torch.bfloat16}
_DT_OF = {torch.float32: F32, torch.bfloat16: BF16, "f32": F32, "bf16": BF16, F32: F32, BF16: BF16}


class SfbDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("B", ctypes.c_int64),
                ("n", ctypes.c_int), ("in_dtype", ctypes.c_int), ("wire_dtype", ctypes.c_int),
                ("out_dtype", ctypes.c_int), ("fuse_sgd", ctypes.c_int), ("lr", ctypes.c_float),
                ("momentum", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("fuse_adam", ctypes.c_int), ("beta1", ctypes.c_float), ("beta2", ctypes.c_float),
                ("eps", ctypes.c_float), ("gather", ctypes.c_int)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("tensor_cores", ctypes.c_int), ("gather_mode", ctypes.c_int),
                ("K", ctypes.c_int64), ("alpha", ctypes.c_float), ("multicast", ctypes.c_int),
                ("recon_bn", ctypes.c_int), ("recon_ctas", ctypes.c_int),
                ("recon_box3d", ctypes.c_int)]


GATHER_NONE, GATHER_NCCL, GATHER_NVLINK_PUSH = 0, 1, 2
GATHER_NAMES = {0: "none", 1: "nccl_allgather", 2: "nvlink_push"}
GATHER_REQ = {"auto": 0, "nccl": 1, "push": 2}          # tag_gather_request_t
COMM_DEFAULT, COMM_NVLS_MULTICAST, COMM_LOOPBACK = 0, 1, 2  # tag_comm_flags_t


class LayerDesc(ctypes.Structure):
    _fields_ = [("M", ctypes.c_int64), ("N", ctypes.c_int64), ("B", ctypes.c_int64),
                ("factor_dtype", ctypes.c_int), ("grad_dtype", ctypes.c_int)]


class Curve(ctypes.Structure):
    _fields_ = [("count", ctypes.c_int), ("bytes", ctypes.POINTER(ctypes.c_uint64)),
                ("ns", ctypes.POINTER(ctypes.c_uint64))]


class ProfiledTopology(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("gather", Curve), ("allreduce", Curve),
                ("tensor_flops", ctypes.c_uint64), ("ps", Curve),
                ("recon_ns", ctypes.POINTER(ctypes.c_uint64)),
                ("local_ns", ctypes.POINTER(ctypes.c_uint64))]


class IlpInstance(ctypes.Structure):
    _fields_ = [("num_ops", ctypes.c_int), ("l", ctypes.c_int), ("g", ctypes.c_int),
                ("op_ns", ctypes.POINTER(ctypes.c_uint64)), ("num_edges", ctypes.c_int),
                ("edge_src", ctypes.POINTER(ctypes.c_int)), ("edge_dst", ctypes.POINTER(ctypes.c_int)),
                ("edge_bytes", ctypes.POINTER(ctypes.c_uint64)), ("grad_bytes", ctypes.c_uint64),
                ("D", ctypes.c_int), ("tau", ctypes.c_uint64)]


class Topology(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("link_bytes_per_s", ctypes.c_uint64),
                ("tensor_flops", ctypes.c_uint64), ("rule", ctypes.c_int)]


_p, _vp, _i, _st = ctypes.POINTER, ctypes.c_void_p, ctypes.c_int, ctypes.c_int
_SIGS = {
    "tag_version": ([], ctypes.c_char_p),
    "tag_status_string": ([_i], ctypes.c_char_p),
    "tag_last_error": ([], ctypes.c_char_p),
    "tag_kernel_launches": ([], ctypes.c_uint64),
    "tag_get_unique_id": ([ctypes.c_char_p], _st),
    "tag_comm_create": ([ctypes.c_char_p, _i, _i, _i, _p(_vp)], _st),
    "tag_comm_create_ex": ([ctypes.c_char_p, _i, _i, _i, ctypes.c_uint, _p(_vp)], _st),
    "tag_comm_destroy": ([_vp], _st),
    "tag_comm_info": ([_vp, _p(_i), _p(_i), _p(_i)], _st),
    "tag_comm_barrier": ([_vp, _vp], _st),
    "tag_sfb_plan": ([_vp, _p(SfbDesc), _p(_vp)], _st),
    "tag_sfb_plan_destroy": ([_vp], _st),
    "tag_sfb_plan_info": ([_vp, _p(PlanInfo)], _st),
    "tag_sfb_sync": ([_vp, _vp, _vp, _vp, _vp], _st),
    "tag_sfb_gather": ([_vp, _vp, _vp, _vp], _st),
    "tag_sfb_reconstruct": ([_vp, _vp, _vp], _st),
    "tag_sfb_bias_grad": ([_vp, _vp, _vp], _st),
    "tag_sfb_sync_sgd": ([_vp, _vp, _vp, _vp, _vp, _vp, _vp], _st),
    "tag_sfb_sync_adam": ([_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp, _vp], _st),
    "tag_sfb_sync_host": ([_vp, _vp, _vp, _vp, _vp], _st),
    "tag_sfb_shard_rows": ([_vp, _i, _p(ctypes.c_int64), _p(ctypes.c_int64)], _st),
    "tag_sfb_sync_sharded": ([_vp, _vp, _vp, _vp, _vp], _st),
    "tag_sfb_sync_sharded_sgd": ([_vp, _vp, _vp, _vp, _vp, _vp], _st),
    "tag_sfb_sync_sharded_adam": ([_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp], _st),
    "tag_local_grad": ([_vp, _vp, _vp, _vp, _vp], _st),
    "tag_dense_allreduce": ([_vp, _vp, _vp], _st),
    "tag_ps_sync": ([_vp, _vp, _i, _vp], _st),
    "tag_sgd_step": ([_vp, _vp, _vp, _vp, _vp], _st),
    "tag_adam_step": ([_vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp], _st),
    "tag_sfb_select": ([_p(LayerDesc), _i, _p(Topology), _p(_i)], _st),
    "tag_sfb_select_profiled": ([_p(LayerDesc), _i, _p(ProfiledTopology), _p(_i)], _st),
    "tag_sfb_ilp_solve": ([_p(IlpInstance), _p(ctypes.c_uint8), _p(ctypes.c_double)], _st),
    "tag_sfb_group_create": ([_p(_vp), _i, _p(_vp)], _st),
    "tag_sfb_group_destroy": ([_vp], _st),
    "tag_sfb_group_sync_sharded": ([_vp, _p(_vp), _p(_vp), _p(_vp), _vp], _st),
    "tag_sfb_group_sync": ([_vp, _p(_vp), _p(_vp), _p(_vp), _vp], _st),
    "tag_sfb_group_gather": ([_vp, _p(_vp), _p(_vp), _vp], _st),
    "tag_sfb_group_sync_sgd": ([_vp, _p(_vp), _p(_vp), _p(_vp), _p(_vp), _p(_vp), _vp], _st),
    "tag_sfb_group_sync_adam": ([_vp, _p(_vp), _p(_vp), _p(_vp), _p(_vp), _p(_vp), ctypes.c_int64,
                                 _p(_vp), _vp], _st),
    "tag_sfb_group_reconstruct": ([_vp, _p(_vp), _vp], _st),
    "tag_sfb_group_bias_grad": ([_vp, _p(_vp), _vp], _st),
}
for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(_lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res
EXPORTS = tuple(_SIGS)


class TagError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        detail = _lib.tag_last_error().decode(errors="replace")
        name = _lib.tag_status_string(status).decode()
        super().__init__(f"{where}: {name}: {detail}")


def _check(st, where):
    if st != OK:
        raise TagError(st, where)


def version():
    return _lib.tag_version().decode()


def kernel_launches():
    """libtag kernels launched by this process so far."""
    return int(_lib.tag_kernel_launches())


def _stream(stream):
    if stream is None:
        return _vp(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return _vp(stream)
    return _vp(stream.cuda_stream)


def _dev(t, dtype, shape, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return _vp(t.data_ptr())


def _host(t, dtype, shape, name):
    if not isinstance(t, torch.Tensor) or t.is_cuda:
        raise TypeError(f"{name} must be a host (CPU) tensor")
    if t.dtype != dtype or tuple(t.shape) != tuple(shape) or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)}")
    return _vp(t.data_ptr())


def unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(_lib.tag_get_unique_id(buf), "tag_get_unique_id")
    return buf.raw


class Comm:
    """One process per GPU. nranks == 1 needs no id (no NCCL communicator is created unless
    loopback=True: a real one-rank NCCL communicator, so every collective code path runs at n = 1).
    multicast=True asks for NVLS multicast stores in the fused push (TAG_COMM_NVLS_MULTICAST)."""

    def __init__(self, nranks, rank, device, uid=None, multicast=False, loopback=False):
        h = _vp()
        idbuf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
        flags = (COMM_NVLS_MULTICAST if multicast else 0) | (COMM_LOOPBACK if loopback else 0)
        _check(_lib.tag_comm_create_ex(idbuf, nranks, rank, device, flags, ctypes.byref(h)),
               "tag_comm_create_ex")
        self._h = h
        self.nranks, self.rank, self.device = nranks, rank, device
        self.loopback = bool(loopback and nranks == 1)

    @classmethod
    def loopback_comm(cls, device=0):
        """One-rank comm with a real NCCL communicator (TAG_COMM_LOOPBACK)."""
        return cls(1, 0, device, loopback=True)

    @property
    def handle(self):
        return self._h

    def barrier(self, stream=None):
        """Stream-ordered device-side barrier of all ranks (no-op for one rank)."""
        _check(_lib.tag_comm_barrier(self._h, _stream(stream)), "tag_comm_barrier")

    def close(self):
        if self._h:
            _check(_lib.tag_comm_destroy(self._h), "tag_comm_destroy")
            self._h = None


class SfbPlan:
    """One replicated Dense layer W (M x N), B rows per replica, n replicas (= comm size)."""

    def __init__(self, comm, M, N, B, in_dtype="bf16", wire_dtype="bf16", out_dtype="f32",
                 fuse_sgd=False, lr=0.0, momentum=0.0, weight_decay=0.0, fuse_adam=False,
                 beta1=0.9, beta2=0.999, eps=1e-8, gather="auto"):
        self.comm = comm
        self.M, self.N, self.B, self.n = M, N, B, comm.nranks
        self.in_dtype, self.wire_dtype, self.out_dtype = (_DT_OF[in_dtype], _DT_OF[wire_dtype],
                                                          _DT_OF[out_dtype])
        d = SfbDesc(M, N, B, comm.nranks, self.in_dtype, self.wire_dtype, self.out_dtype,
                    1 if fuse_sgd else 0, lr, momentum, weight_decay, 1 if fuse_adam else 0,
                    beta1, beta2, eps, GATHER_REQ[gather])
        h = _vp()
        _check(_lib.tag_sfb_plan(comm.handle, ctypes.byref(d), ctypes.byref(h)), "tag_sfb_plan")
        self._h = h

    def _dev(self, t, dtype, shape, name):
        ptr = _dev(t, dtype, shape, name)
        if t.device.index != self.comm.device:
            raise ValueError(f"{name} is on {t.device}, the plan's communicator uses "
                             f"cuda:{self.comm.device}")
        return ptr

    def info(self):
        i = PlanInfo()
        _check(_lib.tag_sfb_plan_info(self._h, ctypes.byref(i)), "tag_sfb_plan_info")
        return {"tensor_cores": bool(i.tensor_cores), "gather": GATHER_NAMES[i.gather_mode],
                "K": int(i.K), "alpha": float(i.alpha), "multicast": bool(i.multicast),
                "recon_bn": int(i.recon_bn), "recon_ctas": int(i.recon_ctas),
                "recon_box3d": bool(i.recon_box3d)}

    # dtypes as torch dtypes
    @property
    def in_torch(self):
        return _TORCH_DT[self.in_dtype]

    @property
    def out_torch(self):
        return _TORCH_DT[self.out_dtype]

    def _xy(self, X, dY):
        return (self._dev(X, self.in_torch, (self.B, self.M), "X"),
                self._dev(dY, self.in_torch, (self.B, self.N), "dY"))

    def sync(self, X, dY, dW, stream=None):
        x, dy = self._xy(X, dY)
        _check(_lib.tag_sfb_sync(self._h, x, dy, self._dev(dW, self.out_torch, (self.M, self.N), "dW"),
                                 _stream(stream)), "tag_sfb_sync")
        return dW

    def gather(self, X, dY, stream=None):
        x, dy = self._xy(X, dY)
        _check(_lib.tag_sfb_gather(self._h, x, dy, _stream(stream)), "tag_sfb_gather")

    def reconstruct(self, dW, stream=None):
        _check(_lib.tag_sfb_reconstruct(self._h, self._dev(dW, self.out_torch, (self.M, self.N), "dW"),
                                        _stream(stream)), "tag_sfb_reconstruct")
        return dW

    def bias_grad(self, db, stream=None):
        """db <- alpha * column sums of the dY_all of this plan's latest synchronisation."""
        _check(_lib.tag_sfb_bias_grad(self._h, self._dev(db, self.out_torch, (self.N,), "db"),
                                      _stream(stream)), "tag_sfb_bias_grad")
        return db

    def sync_sgd(self, X, dY, W, v, dW=None, stream=None):
        x, dy = self._xy(X, dY)
        shape = (self.M, self.N)
        dw = self._dev(dW, self.out_torch, shape, "dW") if dW is not None else _vp()
        _check(_lib.tag_sfb_sync_sgd(self._h, x, dy, self._dev(W, torch.float32, shape, "W"),
                                     self._dev(v, torch.float32, shape, "v"), dw, _stream(stream)),
               "tag_sfb_sync_sgd")

    def sync_adam(self, X, dY, W, m, v, step, dW=None, stream=None):
        """tag_sfb_sync with Adam fused into the epilogue (step >= 1)."""
        x, dy = self._xy(X, dY)
        shape = (self.M, self.N)
        dw = self._dev(dW, self.out_torch, shape, "dW") if dW is not None else _vp()
        _check(_lib.tag_sfb_sync_adam(self._h, x, dy, self._dev(W, torch.float32, shape, "W"),
                                      self._dev(m, torch.float32, shape, "m"),
                                      self._dev(v, torch.float32, shape, "v"), step, dw,
                                      _stream(stream)), "tag_sfb_sync_adam")

    def adam_step(self, dW, W, m, v, step, stream=None):
        shape = (self.M, self.N)
        _check(_lib.tag_adam_step(self._h, self._dev(dW, torch.float32, shape, "dW"),
                                  self._dev(W, torch.float32, shape, "W"), self._dev(m, torch.float32, shape, "m"),
                                  self._dev(v, torch.float32, shape, "v"), step, _stream(stream)),
               "tag_adam_step")

    def shard_rows(self, rank=None):
        """(row_begin, row_count) of `rank`'s dW shard (default: this rank)."""
        b, c = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.tag_sfb_shard_rows(self._h, self.comm.rank if rank is None else rank,
                                       ctypes.byref(b), ctypes.byref(c)), "tag_sfb_shard_rows")
        return b.value, c.value

    def sync_sharded(self, X, dY, dW_shard, stream=None):
        x, dy = self._xy(X, dY)
        _, rc = self.shard_rows()
        dw = self._dev(dW_shard, self.out_torch, (rc, self.N), "dW_shard") if rc > 0 else _vp()
        _check(_lib.tag_sfb_sync_sharded(self._h, x, dy, dw, _stream(stream)),
               "tag_sfb_sync_sharded")
        return dW_shard

    def sync_sharded_sgd(self, X, dY, W, v_shard, stream=None):
        """Sharded SGD-momentum on this rank's rows of W (momentum rows v_shard), then the W
        all-gather: W (M x N fp32) is the whole updated parameter on every rank afterwards."""
        x, dy = self._xy(X, dY)
        _, rc = self.shard_rows()
        v = self._dev(v_shard, torch.float32, (rc, self.N), "v_shard") if rc > 0 else _vp()
        _check(_lib.tag_sfb_sync_sharded_sgd(self._h, x, dy,
                                             self._dev(W, torch.float32, (self.M, self.N), "W"), v,
                                             _stream(stream)), "tag_sfb_sync_sharded_sgd")

    def sync_sharded_adam(self, X, dY, W, m_shard, v_shard, step, stream=None):
        """Sharded Adam on this rank's rows of W (moment rows m_shard, v_shard), then the W
        all-gather."""
        x, dy = self._xy(X, dY)
        _, rc = self.shard_rows()
        m = self._dev(m_shard, torch.float32, (rc, self.N), "m_shard") if rc > 0 else _vp()
        v = self._dev(v_shard, torch.float32, (rc, self.N), "v_shard") if rc > 0 else _vp()
        _check(_lib.tag_sfb_sync_sharded_adam(self._h, x, dy,
                                              self._dev(W, torch.float32, (self.M, self.N), "W"), m, v,
                                              step, _stream(stream)), "tag_sfb_sync_sharded_adam")

    def sync_host(self, X_host, dY_host, dW_host, stream=None):
        _check(_lib.tag_sfb_sync_host(
            self._h, _host(X_host, self.in_torch, (self.B, self.M), "X_host"),
            _host(dY_host, self.in_torch, (self.B, self.N), "dY_host"),
            _host(dW_host, self.out_torch, (self.M, self.N), "dW_host"), _stream(stream)),
            "tag_sfb_sync_host")
        return dW_host

    def local_grad(self, X, dY, dW, stream=None):
        x, dy = self._xy(X, dY)
        _check(_lib.tag_local_grad(self._h, x, dy, self._dev(dW, self.out_torch, (self.M, self.N), "dW"),
                                   _stream(stream)), "tag_local_grad")
        return dW

    def dense_allreduce(self, dW, stream=None):
        _check(_lib.tag_dense_allreduce(self._h, self._dev(dW, self.out_torch, (self.M, self.N), "dW"),
                                        _stream(stream)), "tag_dense_allreduce")
        return dW

    def ps_sync(self, dW, root, stream=None):
        """Replicate-with-PS: reduce to `root` (PreMulSum 1/(nB)) and broadcast back, in place."""
        _check(_lib.tag_ps_sync(self._h, self._dev(dW, self.out_torch, (self.M, self.N), "dW"), root,
                                _stream(stream)), "tag_ps_sync")
        return dW

    def sgd_step(self, dW, W, v, stream=None):
        shape = (self.M, self.N)
        _check(_lib.tag_sgd_step(self._h, self._dev(dW, torch.float32, shape, "dW"),
                                 self._dev(W, torch.float32, shape, "W"),
                                 self._dev(v, torch.float32, shape, "v"), _stream(stream)),
               "tag_sgd_step")

    def close(self):
        if self._h:
            _check(_lib.tag_sfb_plan_destroy(self._h), "tag_sfb_plan_destroy")
            self._h = None


class SfbGroup:
    """A bucket of plans synchronised by one push kernel and one reconstruction launch."""

    def __init__(self, plans):
        self.plans = list(plans)
        arr = (_vp * len(self.plans))(*[p._h for p in self.plans])
        h = _vp()
        _check(_lib.tag_sfb_group_create(arr, len(self.plans), ctypes.byref(h)),
               "tag_sfb_group_create")
        self._h = h

    def _ptrs(self, ts, which):
        out = []
        for p, t in zip(self.plans, ts):
            if which == "X":
                out.append(self.plans[0]._dev(t, p.in_torch, (p.B, p.M), "X"))
            elif which == "dY":
                out.append(self.plans[0]._dev(t, p.in_torch, (p.B, p.N), "dY"))
            else:
                out.append(self.plans[0]._dev(t, p.out_torch, (p.M, p.N), "dW"))
        assert len(out) == len(self.plans), f"{which}: one tensor per plan"
        return (_vp * len(out))(*out)

    def sync(self, Xs, dYs, dWs, stream=None):
        _check(_lib.tag_sfb_group_sync(self._h, self._ptrs(Xs, "X"), self._ptrs(dYs, "dY"),
                                       self._ptrs(dWs, "dW"), _stream(stream)), "tag_sfb_group_sync")

    def sync_sharded(self, Xs, dYs, dW_shards, stream=None):
        ptrs = []
        for p, t in zip(self.plans, dW_shards):
            _, rc = p.shard_rows()
            ptrs.append(self.plans[0]._dev(t, p.out_torch, (rc, p.N), "dW_shard") if rc > 0 else _vp())
        _check(_lib.tag_sfb_group_sync_sharded(self._h, self._ptrs(Xs, "X"), self._ptrs(dYs, "dY"),
                                               (_vp * len(ptrs))(*ptrs), _stream(stream)),
               "tag_sfb_group_sync_sharded")

    def sync_sgd(self, Xs, dYs, Ws, vs, dWs=None, stream=None):
        shapes = [(p.M, p.N) for p in self.plans]
        W = (_vp * len(self.plans))(*[self.plans[0]._dev(w, torch.float32, s, "W") for w, s in zip(Ws, shapes)])
        v = (_vp * len(self.plans))(*[self.plans[0]._dev(x, torch.float32, s, "v") for x, s in zip(vs, shapes)])
        dW = self._ptrs(dWs, "dW") if dWs is not None else None
        _check(_lib.tag_sfb_group_sync_sgd(self._h, self._ptrs(Xs, "X"), self._ptrs(dYs, "dY"), W,
                                           v, dW, _stream(stream)), "tag_sfb_group_sync_sgd")

    def sync_adam(self, Xs, dYs, Ws, ms, vs, step, dWs=None, stream=None):
        shapes = [(p.M, p.N) for p in self.plans]
        arr = lambda ts, nm: (_vp * len(self.plans))(*[self.plans[0]._dev(t, torch.float32, s_, nm)   # noqa: E731
                                                      for t, s_ in zip(ts, shapes)])
        dW = self._ptrs(dWs, "dW") if dWs is not None else None
        _check(_lib.tag_sfb_group_sync_adam(self._h, self._ptrs(Xs, "X"), self._ptrs(dYs, "dY"),
                                            arr(Ws, "W"), arr(ms, "m"), arr(vs, "v"), step, dW,
                                            _stream(stream)), "tag_sfb_group_sync_adam")

    def gather(self, Xs, dYs, stream=None):
        _check(_lib.tag_sfb_group_gather(self._h, self._ptrs(Xs, "X"), self._ptrs(dYs, "dY"),
                                         _stream(stream)), "tag_sfb_group_gather")

    def reconstruct(self, dWs, stream=None):
        _check(_lib.tag_sfb_group_reconstruct(self._h, self._ptrs(dWs, "dW"), _stream(stream)),
               "tag_sfb_group_reconstruct")

    def bias_grad(self, dbs, stream=None):
        ptrs = [self.plans[0]._dev(t, p.out_torch, (p.N,), "db") for p, t in zip(self.plans, dbs)]
        assert len(ptrs) == len(self.plans), "db: one tensor per plan"
        _check(_lib.tag_sfb_group_bias_grad(self._h, (_vp * len(ptrs))(*ptrs), _stream(stream)),
               "tag_sfb_group_bias_grad")

    def close(self):
        if self._h:
            _check(_lib.tag_sfb_group_destroy(self._h), "tag_sfb_group_destroy")
            self._h = None


def select(layers, n, link_bytes_per_s=900_000_000_000, tensor_flops=0, rule=RULE_NORTHSTAR):
    """Per-layer choice (SYNC_SFB / SYNC_ALLREDUCE / SYNC_NONE). layers: iterable of dicts with
    M, N, B and optional factor_dtype / grad_dtype ("bf16" | "f32")."""
    layers = list(layers)
    arr = (LayerDesc * max(1, len(layers)))()
    for i, L in enumerate(layers):
        arr[i] = LayerDesc(L["M"], L["N"], L["B"], _DT_OF[L.get("factor_dtype", "bf16")],
                           _DT_OF[L.get("grad_dtype", "f32")])
    topo = Topology(n, link_bytes_per_s, tensor_flops, rule)
    out = (ctypes.c_int * max(1, len(layers)))()
    _check(_lib.tag_sfb_select(arr, len(layers), ctypes.byref(topo), out), "tag_sfb_select")
    return [out[i] for i in range(len(layers))]


def _curve(points):
    pts = list(points)
    b = (ctypes.c_uint64 * len(pts))(*[int(p[0]) for p in pts])
    t = (ctypes.c_uint64 * len(pts))(*[int(p[1]) for p in pts])
    return Curve(len(pts), b, t), (b, t)


def select_profiled(layers, n, gather_points, allreduce_points, tensor_flops=0, ps_points=None,
                    recon_ns=None, local_ns=None):
    """Per-layer choice from measured cost curves [(bytes, ns), ...] (tag_sfb_select_profiled);
    ps_points (optional) adds the Replicate-with-PS option (SYNC_PS); recon_ns / local_ns
    (optional, per layer) are measured op times replacing the tensor_flops model."""
    layers = list(layers)
    arr = (LayerDesc * max(1, len(layers)))()
    for i, L in enumerate(layers):
        arr[i] = LayerDesc(L["M"], L["N"], L["B"], _DT_OF[L.get("factor_dtype", "bf16")],
                           _DT_OF[L.get("grad_dtype", "f32")])
    g, keep_g = _curve(gather_points)
    a, keep_a = _curve(allreduce_points)
    if ps_points:
        ps, keep_p = _curve(ps_points)
    else:
        ps, keep_p = Curve(0, None, None), None
    rn = ln = None
    if recon_ns is not None or local_ns is not None:
        assert recon_ns is not None and local_ns is not None and len(recon_ns) == len(local_ns) == len(layers)
        rn = (ctypes.c_uint64 * max(1, len(layers)))(*[int(x) for x in recon_ns])
        ln = (ctypes.c_uint64 * max(1, len(layers)))(*[int(x) for x in local_ns])
    topo = ProfiledTopology(n, g, a, tensor_flops, ps,
                            ctypes.cast(rn, ctypes.POINTER(ctypes.c_uint64)) if rn else None,
                            ctypes.cast(ln, ctypes.POINTER(ctypes.c_uint64)) if ln else None)
    out = (ctypes.c_int * max(1, len(layers)))()
    _check(_lib.tag_sfb_select_profiled(arr, len(layers), ctypes.byref(topo), out),
           "tag_sfb_select_profiled")
    del keep_g, keep_a, keep_p, rn, ln
    return [out[i] for i in range(len(layers))]


def ilp_solve(inst):
    """General SFB cut ILP (tag_sfb_ilp_solve). inst: dict(num_ops, l, g, op_ns[list], edges
    [(src or -1, dst, bytes)], grad_bytes, D, tau). Returns (alpha list, objective seconds)."""
    V, E = inst["num_ops"], inst["edges"]
    op_ns = (ctypes.c_uint64 * V)(*inst["op_ns"])
    ne = max(1, len(E))
    src = (ctypes.c_int * ne)(*[e[0] for e in E])
    dst = (ctypes.c_int * ne)(*[e[1] for e in E])
    byt = (ctypes.c_uint64 * ne)(*[e[2] for e in E])
    c = IlpInstance(V, inst["l"], inst["g"], op_ns, len(E), src, dst, byt, inst["grad_bytes"],
                    inst["D"], inst["tau"])
    alpha = (ctypes.c_uint8 * V)()
    obj = ctypes.c_double()
    _check(_lib.tag_sfb_ilp_solve(ctypes.byref(c), alpha, ctypes.byref(obj)), "tag_sfb_ilp_solve")
    return [alpha[i] for i in range(V)], obj.value
