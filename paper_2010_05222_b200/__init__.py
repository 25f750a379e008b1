"""B200-native Partial FC (arXiv 2010.05222): thin Python binding over the C-ABI library libpfc.so.

Every step of the hot path runs in the library's CUDA kernels; this module only marshals arguments
(pointers from torch tensors, the CUDA stream, the NCCL unique id broadcast over torch.distributed).
It never falls back to another implementation: if libpfc.so is missing or fails to load, import of
the binding raises.

    from paper_2010_05222_b200 import PartialFC
    pfc = PartialFC(num_classes=10_000_000, dim=512, batch=256, sample_rate=0.1, precision="bf16")
    pfc.forward_backward(x, labels, grad_x, loss)   # x [B, d] fp32 cuda, labels [B] int64 cuda
    pfc.step(lr=0.1)
"""
import ctypes
import os

__all__ = ["PartialFC", "load_library", "unique_id", "group_forward_backward", "sample_shard", "PfcError", "MARGINS",
           "PRECISIONS"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# PFC_LIB: an alternative build of the same library (A/B timing of kernel variants); default the in-tree build
LIB_PATH = os.environ.get("PFC_LIB") or os.path.join(_HERE, "_lib", "libpfc.so")

MARGINS = {"none": 0, "arcface": 1, "cosface": 2}
PRECISIONS = {"fp32": 0, "bf16": 1}
COMM_MODES = {"nccl": 0, "loopback": 1, "nccl_fused": 2, "loopback_fused": 3}
SAMPLE_MODES = {"pprn": 0, "pprn_paper": 1, "random": 2}
STATUS = {0: "PFC_OK", 1: "PFC_ERR_CONFIG", 2: "PFC_ERR_CONTRACT", 3: "PFC_ERR_DATA", 4: "PFC_ERR_DEGENERATE",
          5: "PFC_ERR_NUMERIC", 6: "PFC_ERR_CUDA", 7: "PFC_ERR_NCCL", 8: "PFC_ERR_OOM"}

# Every symbol include/pfc.h declares (checked by tests/test_abi.py).
EXPORTS = ["pfc_get_unique_id", "pfc_init", "pfc_destroy", "pfc_last_error", "pfc_forward_backward",
           "pfc_forward_backward_host", "pfc_step", "pfc_shard_range", "pfc_sizes", "pfc_param_ptrs",
           "pfc_get_sampled", "pfc_get_sampled_grad", "pfc_get_lse", "pfc_get_step", "pfc_set_step", "pfc_check",
           "pfc_launch_count", "pfc_path_flags", "pfc_get_state", "pfc_set_state", "pfc_version", "pfc_group_forward_backward", "pfc_sample_shard",
           "pfc_profile_enable", "pfc_profile_read", "pfc_profile_section", "pfc_train_step", "pfc_train_step_host",
           "pfc_train_step_host_async", "pfc_forward_backward_host_async",
           "pfc_group_train_step", "pfc_get_metrics"]
PROF_SECTIONS = 10


class PfcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


PARAM_LOCATIONS = {"device": 0, "host": 1}


class _Config(ctypes.Structure):
    _fields_ = [("num_classes", ctypes.c_int64), ("dim", ctypes.c_int32), ("batch", ctypes.c_int32),
                ("sample_rate", ctypes.c_double), ("scale", ctypes.c_float), ("margin_type", ctypes.c_int32),
                ("margin", ctypes.c_float), ("momentum", ctypes.c_float), ("weight_decay", ctypes.c_float),
                ("precision", ctypes.c_int32), ("seed", ctypes.c_uint64), ("rank", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("device", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("comm_mode", ctypes.c_int32), ("sample_mode", ctypes.c_int32), ("param_location", ctypes.c_int32),
                ("ignore_index", ctypes.c_int32)]


_lib = None


def load_library(path=LIB_PATH):
    """Load libpfc.so (raises if it is missing: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2010_05222_b200.build` "
                          "(or __graft_entry__.build())")
    lib = ctypes.CDLL(path)
    P, I64, U64, F, VP = ctypes.POINTER, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float, ctypes.c_void_p
    st = ctypes.c_int
    sig = {
        "pfc_get_unique_id": (st, [VP]),
        "pfc_init": (st, [P(_Config), P(VP)]),
        "pfc_destroy": (st, [VP]),
        "pfc_last_error": (ctypes.c_char_p, [VP]),
        "pfc_forward_backward": (st, [VP, VP, VP, VP, VP, VP]),
        "pfc_forward_backward_host": (st, [VP, VP, VP, VP, VP, VP]),
        "pfc_step": (st, [VP, F, VP]),
        "pfc_shard_range": (st, [VP, P(I64), P(I64)]),
        "pfc_sizes": (st, [VP, P(I64), P(I64)]),
        "pfc_param_ptrs": (st, [VP, P(VP), P(VP)]),
        "pfc_get_sampled": (st, [VP, VP, I64, P(I64)]),
        "pfc_get_sampled_grad": (st, [VP, VP, I64]),
        "pfc_get_lse": (st, [VP, VP, I64]),
        "pfc_get_step": (st, [VP, P(U64)]),
        "pfc_set_step": (st, [VP, U64]),
        "pfc_check": (st, [VP]),
        "pfc_launch_count": (I64, [VP]),
        "pfc_path_flags": (ctypes.c_uint32, [VP]),
        "pfc_get_state": (ctypes.c_int, [VP, VP, VP, VP]),
        "pfc_set_state": (ctypes.c_int, [VP, VP, VP, VP]),
        "pfc_version": (ctypes.c_char_p, []),
        "pfc_train_step": (st, [VP, VP, VP, VP, VP, F, VP]),
        "pfc_get_metrics": (st, [VP, P(F), P(F)]),
        "pfc_train_step_host": (st, [VP, VP, VP, VP, VP, F, VP]),
        "pfc_train_step_host_async": (st, [VP, VP, VP, VP, VP, F, VP]),
        "pfc_forward_backward_host_async": (st, [VP, VP, VP, VP, VP, VP]),
        "pfc_group_train_step": (st, [P(VP), ctypes.c_int32, P(VP), P(VP), P(VP), VP, F, VP]),
        "pfc_profile_enable": (st, [VP, ctypes.c_int32]),
        "pfc_profile_read": (st, [VP, P(ctypes.c_double), P(I64)]),
        "pfc_profile_section": (ctypes.c_char_p, [ctypes.c_int32]),
        "pfc_group_forward_backward": (st, [P(VP), ctypes.c_int32, P(VP), P(VP), P(VP), VP, VP]),
        "pfc_sample_shard": (st, [I64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, U64, U64, VP, ctypes.c_int32,
                                  ctypes.c_int32, VP, P(I64), VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


def unique_id():
    """128-byte NCCL unique id (rank 0), to be broadcast to the other ranks."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    s = lib.pfc_get_unique_id(buf)
    if s:
        raise PfcError(s, lib.pfc_last_error(None).decode())
    return bytes(buf.raw)


class _DevArray:
    """Zero-copy torch view of library-owned device memory (via __cuda_array_interface__)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _ptr(t):
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


class PartialFC:
    """One rank of the model-parallel, PPRN-sampled margin-softmax layer (Alg.1 + §3.2.2)."""

    def __init__(self, num_classes, dim, batch, sample_rate=0.1, scale=64.0, margin_type="arcface", margin=0.5,
                 momentum=0.9, weight_decay=0.0, precision="bf16", seed=0, rank=0, world_size=1, device=0,
                 nccl_unique_id=None, comm_mode="nccl", sample_mode="pprn", param_location="device",
                 ignore_index=False):
        self._lib = load_library()
        self.param_location = param_location
        self.rank, self.world_size, self.device = rank, world_size, device
        self.dim, self.batch, self.num_classes = dim, batch, num_classes
        self._id_buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128) if nccl_unique_id else None
        cfg = _Config(num_classes, dim, batch, float(sample_rate), float(scale),
                      MARGINS[margin_type] if isinstance(margin_type, str) else int(margin_type), float(margin),
                      float(momentum), float(weight_decay),
                      PRECISIONS[precision] if isinstance(precision, str) else int(precision), int(seed), rank,
                      world_size, device, ctypes.cast(self._id_buf, ctypes.c_void_p) if self._id_buf else None,
                      COMM_MODES[comm_mode] if isinstance(comm_mode, str) else int(comm_mode),
                      SAMPLE_MODES[sample_mode] if isinstance(sample_mode, str) else int(sample_mode),
                      PARAM_LOCATIONS[param_location], 1 if ignore_index else 0)
        h = ctypes.c_void_p()
        s = self._lib.pfc_init(ctypes.byref(cfg), ctypes.byref(h))
        if s:
            raise PfcError(s, self._lib.pfc_last_error(None).decode())
        self._h = h
        a, n = ctypes.c_int64(), ctypes.c_int64()
        self._lib.pfc_shard_range(h, ctypes.byref(a), ctypes.byref(n))
        self.shard_start, self.shard_size = a.value, n.value
        M, kmax = ctypes.c_int64(), ctypes.c_int64()
        self._lib.pfc_sizes(h, ctypes.byref(M), ctypes.byref(kmax))
        self.global_batch, self.k_max = M.value, kmax.value

    @classmethod
    def from_process_group(cls, group=None, **kw):
        """Create one rank per process: rank 0 makes the NCCL id, torch.distributed broadcasts it."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rank=rank, world_size=world, nccl_unique_id=obj[0] if world > 1 else None, **kw)

    # -------------------------------------------------------------- errors
    def _check(self, s):
        if s:
            raise PfcError(s, self._lib.pfc_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pfc_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -------------------------------------------------------------- hot path
    @staticmethod
    def _stream(stream):
        if stream is None:
            import torch
            stream = torch.cuda.current_stream()
        return ctypes.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))

    def forward_backward(self, x, labels, grad_x, loss=None, stream=None):
        """x [B, d] float32, labels [B] int64, grad_x [B, d] float32 (output), loss [1] float32 or None —
        all CUDA tensors on this rank's device, contiguous."""
        self._check(self._lib.pfc_forward_backward(self._h, _ptr(x), _ptr(labels), _ptr(grad_x), _ptr(loss),
                                                   self._stream(stream)))

    def forward_backward_host(self, x, labels, grad_x, loss=None, stream=None, sync=True):
        """Same with host (ideally pinned) CPU tensors; copies are inside the call; synchronises unless sync=False."""
        fn = self._lib.pfc_forward_backward_host if sync else self._lib.pfc_forward_backward_host_async
        self._check(fn(self._h, _ptr(x), _ptr(labels), _ptr(grad_x), _ptr(loss), self._stream(stream)))

    def train_step(self, x, labels, grad_x, loss=None, lr=0.1, stream=None):
        """forward_backward + step(lr) fused (the SGD update runs in the dW contraction's epilogue)."""
        self._check(self._lib.pfc_train_step(self._h, _ptr(x), _ptr(labels), _ptr(grad_x), _ptr(loss), float(lr),
                                             self._stream(stream)))

    def train_step_host(self, x, labels, grad_x, loss=None, lr=0.1, stream=None, sync=True):
        """train_step with host (pinned) CPU tensors; copies inside the call; synchronises unless sync=False
        (pfc_train_step_host_async: grad_x / loss valid once the stream completes)."""
        fn = self._lib.pfc_train_step_host if sync else self._lib.pfc_train_step_host_async
        self._check(fn(self._h, _ptr(x), _ptr(labels), _ptr(grad_x), _ptr(loss), float(lr), self._stream(stream)))

    def step(self, lr, stream=None):
        self._check(self._lib.pfc_step(self._h, float(lr), self._stream(stream)))

    # -------------------------------------------------------------- state / introspection
    def params(self):
        """(W, V) zero-copy torch views of the library-owned [C_local, d] float32 shards: CUDA tensors, or CPU
        tensors over the page-locked host memory with param_location="host" (synchronise before touching them)."""
        import torch
        W, V = ctypes.c_void_p(), ctypes.c_void_p()
        self._check(self._lib.pfc_param_ptrs(self._h, ctypes.byref(W), ctypes.byref(V)))
        shape = (self.shard_size, self.dim)
        if self.param_location == "host":
            n = self.shard_size * self.dim
            return tuple(torch.frombuffer((ctypes.c_float * n).from_address(p.value), dtype=torch.float32).view(shape)
                         for p in (W, V))
        dev = torch.device("cuda", self.device)
        return (torch.as_tensor(_DevArray(W.value, shape, "<f4"), device=dev),
                torch.as_tensor(_DevArray(V.value, shape, "<f4"), device=dev))

    def sampled(self):
        """Sampled global class ids of the last forward_backward (ascending), as an int64 numpy array."""
        import numpy as np
        k = ctypes.c_int64()
        self._check(self._lib.pfc_get_sampled(self._h, None, 0, ctypes.byref(k)))
        out = np.empty(k.value, dtype=np.int64)
        self._check(self._lib.pfc_get_sampled(self._h, out.ctypes.data_as(ctypes.c_void_p), k.value, ctypes.byref(k)))
        return out

    def sampled_grad(self):
        """[k_i, d] float32 numpy gradient of the loss w.r.t. the raw sampled W rows (before step)."""
        import numpy as np
        k = ctypes.c_int64()
        self._check(self._lib.pfc_get_sampled(self._h, None, 0, ctypes.byref(k)))
        out = np.empty((k.value, self.dim), dtype=np.float32)
        self._check(self._lib.pfc_get_sampled_grad(self._h, out.ctypes.data_as(ctypes.c_void_p), k.value))
        return out

    def metrics(self):
        """(loss, CA_pcc) of the last step (Eq.5, Eq.7); synchronises."""
        L, ca = ctypes.c_float(), ctypes.c_float()
        self._check(self._lib.pfc_get_metrics(self._h, ctypes.byref(L), ctypes.byref(ca)))
        return L.value, ca.value

    def lse(self):
        import numpy as np
        out = np.empty(self.global_batch, dtype=np.float32)
        self._check(self._lib.pfc_get_lse(self._h, out.ctypes.data_as(ctypes.c_void_p), self.global_batch))
        return out

    @property
    def step_count(self):
        v = ctypes.c_uint64()
        self._check(self._lib.pfc_get_step(self._h, ctypes.byref(v)))
        return v.value

    @step_count.setter
    def step_count(self, v):
        self._check(self._lib.pfc_set_step(self._h, int(v)))

    def check(self):
        self._check(self._lib.pfc_check(self._h))

    def get_state(self):
        """Checkpoint: (W, V, step) of this shard as host numpy arrays ([C_local, d] float32) and an int."""
        import numpy as np
        W = np.empty((self.shard_size, self.dim), dtype=np.float32)
        V = np.empty_like(W)
        st = ctypes.c_uint64()
        self._check(self._lib.pfc_get_state(self._h, W.ctypes.data, V.ctypes.data, ctypes.byref(st)))
        return W, V, st.value

    def set_state(self, W=None, V=None, step=None):
        """Resume: load any of W, V ([C_local, d] float32 host arrays) and the step counter."""
        import numpy as np
        ptr = []
        for a in (W, V):
            if a is None:
                ptr.append(None)
            else:
                a = np.ascontiguousarray(a, dtype=np.float32)
                if a.shape != (self.shard_size, self.dim):
                    raise ValueError(f"state array must be {(self.shard_size, self.dim)}, got {a.shape}")
                ptr.append(a)
        st = ctypes.c_uint64(int(step)) if step is not None else None
        self._check(self._lib.pfc_set_state(self._h, ptr[0].ctypes.data if ptr[0] is not None else None,
                                            ptr[1].ctypes.data if ptr[1] is not None else None,
                                            ctypes.byref(st) if st is not None else None))

    def profile(self, enable=True):
        """Record CUDA events between the kernels of every following step (pfc_profile_enable)."""
        self._check(self._lib.pfc_profile_enable(self._h, 1 if enable else 0))

    def profile_read(self):
        """{section: (total_ms, launches)} accumulated since the last read (synchronises)."""
        ms = (ctypes.c_double * PROF_SECTIONS)()
        cnt = (ctypes.c_int64 * PROF_SECTIONS)()
        self._check(self._lib.pfc_profile_read(self._h, ms, cnt))
        return {self._lib.pfc_profile_section(i).decode(): (ms[i], cnt[i]) for i in range(PROF_SECTIONS)}

    def launch_count(self):
        return int(self._lib.pfc_launch_count(self._h))

    PATH_TENSOR_CORES, PATH_FUSED_GATHER, PATH_FUSED_DWX, PATH_EFORM = 1, 2, 4, 8

    def path_flags(self):
        """PFC_PATH_* bits of the kernel path chosen at init (include/pfc.h)."""
        return int(self._lib.pfc_path_flags(self._h))


def _stream_ptr(stream):
    return PartialFC._stream(stream)


def group_forward_backward(ranks, xs, labels, grad_xs, loss=None, stream=None, lr=None):
    """One forward + backward of every rank of a loopback group (PartialFC(..., comm_mode="loopback")); with
    lr given, the fused train step (update applied inside the dW contraction)."""
    lib = load_library()
    n = len(ranks)
    VPA = ctypes.c_void_p * n
    hs = VPA(*[r._h for r in ranks])
    args = (hs, n, VPA(*[t.data_ptr() for t in xs]), VPA(*[t.data_ptr() for t in labels]),
            VPA(*[t.data_ptr() for t in grad_xs]), _ptr(loss))
    if lr is None:
        s = lib.pfc_group_forward_backward(*args, _stream_ptr(stream))
    else:
        s = lib.pfc_group_train_step(*args, float(lr), _stream_ptr(stream))
    if s:
        msg = lib.pfc_last_error(None).decode()
        for r in ranks:
            msg = msg or lib.pfc_last_error(r._h).decode()
        raise PfcError(s, msg)


def sample_shard(num_classes, world_size, rank, sample_rate, seed, step, labels, stream=None, sample_mode="pprn"):
    """Standalone sampler of one shard on the GPU: labels = global-batch int64 CUDA tensor.
    Returns the sampled global ids (ascending) as an int64 CUDA tensor."""
    import torch
    lib = load_library()
    base, extra = divmod(num_classes, world_size)
    C_local = base + (1 if rank < extra else 0)
    import math
    k_max = min(C_local, int(math.ceil(float(sample_rate) * float(C_local))) + 1 + min(labels.numel(), C_local))
    out = torch.empty(max(k_max, 1), dtype=torch.int64, device=labels.device)
    k = ctypes.c_int64()
    s = lib.pfc_sample_shard(num_classes, world_size, rank, float(sample_rate), int(seed), int(step),
                             _ptr(labels), labels.numel(),
                             SAMPLE_MODES[sample_mode] if isinstance(sample_mode, str) else int(sample_mode),
                             _ptr(out), ctypes.byref(k), _stream_ptr(stream))
    if s:
        raise PfcError(s, lib.pfc_last_error(None).decode())
    return out[:k.value]
