"""Thin ctypes binding of libmel (include/mel.h).  Argument marshalling only:
every step of the method runs in the library's CUDA kernels.  There is no CPU
fallback: if libmel.so is missing or fails to load this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field as dc_field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmel.so")
# A/B comparisons of two builds (tools/ab_bench.sh): MEL_LIB names another in-tree build
if os.environ.get("MEL_LIB"):
    LIB_PATH = os.path.join(os.path.dirname(LIB_PATH), os.path.basename(os.environ["MEL_LIB"]))

OK, EAGAIN, EOS = 0, 1, 2
EINVAL, ECLOSED, EPROTO, ECUDA, ENCCL, ENOMEM, ENONFINITE = -1, -2, -3, -4, -5, -6, -7
FP32, BF16 = 0, 1
STORE_F32, STORE_BF16 = 0, 1
FLAG_TIMING = 1
FLAG_NO_ZERO = 2
FLAG_UNFUSED_ADAM = 8
FLAG_NCCL_EXCHANGE = 16
FLAG_FP32_EXCHANGE = 32
K_COMMIT, K_SAMPLE, K_GATHER, K_HEAD_FWD, K_OUT_FWD_DW, K_OUT_DH, K_HEAD_BWD, K_ALLREDUCE, K_ADAM, K_LOSS = range(10)
KERNEL_NAMES = ["commit", "sample", "gather", "head_fwd", "out_fwd_dw", "out_dh", "head_bwd", "allreduce",
                "adam", "loss"]
ABI_VERSION = 2
RESERVOIR, FIFO, FIRO = 0, 1, 2

EXPORTS = ["mel_config_default", "mel_nccl_unique_id", "mel_create", "mel_destroy", "mel_last_error",
           "mel_param_layout", "mel_set_params", "mel_get_params", "mel_get_state", "mel_set_state",
           "reservoir_put", "reservoir_close", "reservoir_sample_batch", "surrogate_step", "surrogate_step_result",
           "surrogate_eval",
           "reservoir_stats", "reservoir_dump", "mel_sync", "mel_kernel_time", "mel_kernel_time_reset",
           "mel_launch_count", "mel_set_flags", "mel_debug_counters", "reservoir_ingest",
           "surrogate_train_offline", "reservoir_put_generated", "mel_params_copy", "mel_create_virtual",
           "surrogate_step_virtual", "mel_stream_wait_event", "reservoir_checkpoint_bytes", "reservoir_save",
           "reservoir_load"]
# include/mel_heat.h (on-device heat-equation client)
HEAT_EXPORTS = ["mel_heat_create", "mel_heat_basis_bytes", "mel_heat_grid", "mel_heat_tau", "mel_heat_fields",
                "mel_heat_destroy"]
# include/mel_dataset.h (offline baseline data path; host code in libmel.so)
DATASET_EXPORTS = ["mel_dataset_create", "mel_dataset_append", "mel_dataset_finish", "mel_dataset_open",
                   "mel_dataset_count", "mel_dataset_n_field", "mel_dataset_epoch_order", "mel_dataset_read",
                   "mel_dataset_close"]
# include/mel_ingest.h (host-only ingest channel; in libmel.so and libmel_ingest.so)
INGEST_EXPORTS = ["mel_ingest_create", "mel_ingest_next", "mel_ingest_release", "mel_ingest_outstanding",
                  "mel_ingest_stats_get", "mel_ingest_segment", "mel_ingest_destroy", "mel_client_open",
                  "mel_client_send", "mel_client_finalize", "mel_client_close", "mel_route"]
INGEST_LIB_PATH = os.path.join(HERE, "libmel_ingest.so")


class MelError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("libmel error %d: %s" % (code, msg))
        self.code = code


class _Config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("n_field", C.c_uint32), ("hidden", C.c_uint32 * 2),
                ("capacity", C.c_uint32), ("threshold", C.c_uint32), ("batch", C.c_uint32),
                ("steps_per_sim", C.c_uint32), ("temp_lo", C.c_float), ("temp_hi", C.c_float),
                ("precision", C.c_uint32), ("storage", C.c_uint32), ("lr0", C.c_double), ("lr_min", C.c_double),
                ("lr_halving_samples", C.c_uint64), ("beta1", C.c_double), ("beta2", C.c_double),
                ("eps", C.c_double), ("seed", C.c_uint64), ("staging_entries", C.c_uint32), ("flags", C.c_uint32),
                ("policy", C.c_uint32), ("pad", C.c_uint32)]


class _Stats(C.Structure):
    _fields_ = [("population", C.c_uint64), ("unseen", C.c_uint64), ("seen", C.c_uint64), ("puts", C.c_uint64),
                ("committed", C.c_uint64), ("draws", C.c_uint64), ("evictions", C.c_uint64),
                ("pending", C.c_uint64), ("steps", C.c_uint64), ("samples", C.c_uint64),
                ("hist", C.c_uint64 * 64), ("over", C.c_uint32), ("closed", C.c_uint32), ("last_loss", C.c_double)]


class _StateView(C.Structure):
    _fields_ = [("p", C.POINTER(C.c_void_p)), ("m", C.POINTER(C.c_void_p)), ("v", C.POINTER(C.c_void_p)),
                ("adam_step", C.c_uint64), ("samples_seen", C.c_uint64)]


class _IngestMsg(C.Structure):
    _fields_ = [("sim_id", C.c_uint32), ("t", C.c_uint32), ("X", C.c_float * 5), ("pad", C.c_uint32),
                ("field", C.POINTER(C.c_float)), ("ticket", C.c_uint64)]


class _IngestStats(C.Structure):
    _fields_ = [("received", C.c_uint64), ("duplicates", C.c_uint64), ("abandoned", C.c_uint64),
                ("finalized", C.c_uint64), ("clients", C.c_uint64), ("bytes", C.c_uint64)]


def _ingest_sigs():
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    return {
        "mel_ingest_create": (C.c_int, [C.c_char_p, u32, u32, u32, u32, C.POINTER(vp)]),
        "mel_ingest_next": (C.c_int, [vp, C.POINTER(_IngestMsg), u32]),
        "mel_ingest_release": (C.c_int, [vp]),
        "mel_ingest_outstanding": (u32, [vp]),
        "mel_ingest_stats_get": (C.c_int, [vp, C.POINTER(_IngestStats)]),
        "mel_ingest_segment": (C.c_int, [vp, C.POINTER(vp), C.POINTER(u64)]),
        "mel_ingest_destroy": (None, [vp]),
        "mel_client_open": (C.c_int, [C.c_char_p, u32, u32, C.POINTER(vp)]),
        "mel_client_send": (C.c_int, [vp, u32, C.POINTER(C.c_float), C.POINTER(C.c_double), u32]),
        "mel_client_finalize": (C.c_int, [vp, u32]),
        "mel_client_close": (None, [vp]),
        "mel_route": (u32, [u32, u32, u32]),
    }


def _bind(lib, sig):
    for name, (res, args) in sig.items():
        if os.environ.get("MEL_LIB") and not hasattr(lib, name):
            continue                     # an older A/B build without this entry point
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


_lib = None
_ingest_lib = None


def load_ingest_library(path: str = INGEST_LIB_PATH):
    """libmel_ingest.so: the clients' side of the ingest channel (host code only, no CUDA)."""
    global _ingest_lib
    if _ingest_lib is not None:
        return _ingest_lib
    if not os.path.exists(path):
        raise OSError("libmel_ingest.so not built at %s (run python -m paper_2309_16743_b200.build)" % path)
    lib = C.CDLL(path)
    _bind(lib, _ingest_sigs())
    _ingest_lib = lib
    return lib


def load_library(path: str = LIB_PATH):
    """Load libmel.so (raises OSError if absent: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise OSError("libmel.so not built at %s (run python -m paper_2309_16743_b200.build)" % path)
    lib = C.CDLL(path)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32
    sig = {
        "mel_config_default": (C.c_int, [C.POINTER(_Config), u32, u32]),
        "mel_nccl_unique_id": (C.c_int, [vp]),
        "mel_create": (C.c_int, [C.POINTER(_Config), C.c_int, C.c_int, vp, C.c_int, vp, C.POINTER(vp)]),
        "mel_destroy": (None, [vp]),
        "mel_last_error": (C.c_char_p, [vp]),
        "mel_param_layout": (C.c_int, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u64)]),
        "mel_set_params": (C.c_int, [vp, C.POINTER(vp)]),
        "mel_get_params": (C.c_int, [vp, C.POINTER(vp)]),
        "mel_get_state": (C.c_int, [vp, C.POINTER(_StateView)]),
        "mel_set_state": (C.c_int, [vp, C.POINTER(_StateView)]),
        "reservoir_put": (C.c_int, [vp, u32, u32, C.POINTER(C.c_float), vp, C.c_int]),
        "reservoir_close": (C.c_int, [vp]),
        "reservoir_sample_batch": (C.c_int, [vp, C.POINTER(i32), C.POINTER(u32)]),
        "surrogate_step": (C.c_int, [vp, C.POINTER(C.c_double)]),
        "surrogate_step_result": (C.c_int, [vp, u64, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
        "surrogate_eval": (C.c_int, [vp, C.POINTER(C.c_float), C.POINTER(u32), C.POINTER(C.c_float), u32,
                                     C.POINTER(C.c_double), C.POINTER(C.c_float)]),
        "reservoir_stats": (C.c_int, [vp, C.POINTER(_Stats)]),
        "reservoir_dump": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),
        "mel_sync": (C.c_int, [vp]),
        "mel_kernel_time": (C.c_int, [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(u64)]),
        "mel_kernel_time_reset": (C.c_int, [vp]),
        "mel_launch_count": (C.c_int, [vp, C.POINTER(u64)]),
        "mel_set_flags": (C.c_int, [vp, u32]),
        "mel_debug_counters": (C.c_int, [vp, C.POINTER(u64), C.c_int]),
        "reservoir_ingest": (C.c_int, [vp, vp, u32, u32, C.POINTER(u32)]),
        "surrogate_train_offline": (C.c_int, [vp, vp, u64, u32, u32, u32, C.POINTER(C.c_double), C.POINTER(u32)]),
        "mel_dataset_create": (C.c_int, [C.c_char_p, u32, C.POINTER(vp)]),
        "mel_dataset_append": (C.c_int, [vp, u32, u32, C.POINTER(C.c_float), C.POINTER(C.c_float)]),
        "mel_dataset_finish": (C.c_int, [vp]),
        "mel_dataset_open": (C.c_int, [C.c_char_p, u32, C.POINTER(vp)]),
        "mel_dataset_count": (u64, [vp]),
        "mel_dataset_n_field": (u32, [vp]),
        "mel_dataset_epoch_order": (C.c_int, [u64, u64, u32, C.POINTER(u32)]),
        "mel_dataset_read": (C.c_int, [vp, C.POINTER(u32), u32, C.POINTER(u32), C.POINTER(u32), C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), u64]),
        "mel_dataset_close": (None, [vp]),
        "mel_params_copy": (C.c_int, [vp, vp]),
        "mel_stream_wait_event": (C.c_int, [vp, vp]),
        "reservoir_checkpoint_bytes": (C.c_int, [vp, C.POINTER(u64)]),
        "reservoir_save": (C.c_int, [vp, vp]),
        "reservoir_load": (C.c_int, [vp, vp]),
        "mel_create_virtual": (C.c_int, [C.POINTER(_Config), C.c_int, C.c_int, vp, C.POINTER(vp)]),
        "surrogate_step_virtual": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(C.c_double)]),
        "reservoir_put_generated": (C.c_int, [vp, vp, C.POINTER(u32), C.POINTER(C.c_float), C.POINTER(u32), u32,
                                              C.POINTER(u32)]),
        "mel_heat_create": (C.c_int, [u32, u32, C.c_double, C.c_double, C.c_double, C.POINTER(vp)]),
        "mel_heat_basis_bytes": (u64, [vp]),
        "mel_heat_grid": (u32, [vp]),
        "mel_heat_tau": (u32, [vp]),
        "mel_heat_fields": (C.c_int, [vp, vp, vp, u32, vp, vp]),
        "mel_heat_destroy": (None, [vp]),
    }
    sig.update(_ingest_sigs())
    _bind(lib, sig)
    _lib = lib
    return lib


@dataclass
class Config:
    n_field: int
    hidden: tuple = (256, 256)
    capacity: int = 6000
    threshold: int = 1000
    batch: int = 10
    steps_per_sim: int = 100
    temp_lo: float = 100.0
    temp_hi: float = 500.0
    precision: int = FP32
    storage: int = STORE_F32
    lr0: float = 1e-3
    lr_min: float = 2.5e-4
    lr_halving_samples: int = 10000
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 1
    staging_entries: int = 16
    flags: int = 0
    policy: int = RESERVOIR

    def to_c(self) -> _Config:
        c = _Config()
        c.abi_version = ABI_VERSION
        c.n_field = self.n_field
        h = list(self.hidden) + [0, 0]
        c.hidden[0], c.hidden[1] = h[0], h[1]
        for k in ("capacity", "threshold", "batch", "steps_per_sim", "temp_lo", "temp_hi", "precision", "storage",
                  "lr0", "lr_min", "lr_halving_samples", "beta1", "beta2", "eps", "seed", "staging_entries", "flags",
                  "policy"):
            setattr(c, k, getattr(self, k))
        return c


def nccl_unique_id() -> bytes:
    lib = load_library()
    buf = C.create_string_buffer(128)
    r = lib.mel_nccl_unique_id(buf)
    if r != OK:
        raise MelError(r, "ncclGetUniqueId failed")
    return buf.raw


def _fptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Context:
    """One rank's trainer + reservoir.  `device` is the CUDA ordinal; `stream` an
    optional cudaStream_t handle (int)."""

    def __init__(self, cfg: Config, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 device: int = 0, stream: int | None = None):
        self.lib = load_library()
        self.cfg = cfg
        self._c = cfg.to_c()
        self._stream = stream
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        r = self.lib.mel_create(C.byref(self._c), rank, world, idbuf, device, C.c_void_p(stream) if stream else None,
                                C.byref(h))
        if r != OK:
            raise MelError(r, "mel_create failed (see stderr)")
        self.h = h
        n = C.c_uint32()
        shapes = (C.c_uint32 * 12)()
        tot = C.c_uint64()
        self.lib.mel_param_layout(self.h, C.byref(n), shapes, C.byref(tot))
        self.shapes = [(shapes[2 * i], shapes[2 * i + 1]) for i in range(n.value)]
        self.n_params = tot.value

    @classmethod
    def _from_handle(cls, cfg: Config, h, lib):
        self = cls.__new__(cls)
        self.lib, self.cfg, self._c, self.h = lib, cfg, cfg.to_c(), h
        self._stream = None
        n = C.c_uint32()
        shapes = (C.c_uint32 * 12)()
        tot = C.c_uint64()
        lib.mel_param_layout(h, C.byref(n), shapes, C.byref(tot))
        self.shapes = [(shapes[2 * i], shapes[2 * i + 1]) for i in range(n.value)]
        self.n_params = tot.value
        return self

    # -- lifecycle -------------------------------------------------------------------
    def close_ctx(self):
        if getattr(self, "h", None):
            self.lib.mel_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close_ctx()
        except Exception:
            pass

    def _check(self, r, allowed=(OK,)):
        if r in allowed:
            return r
        msg = self.lib.mel_last_error(self.h).decode(errors="replace") if self.h else ""
        raise MelError(r, msg)

    # -- reservoir ---------------------------------------------------------------------
    def put(self, sim: int, t: int, X, field, zero_copy: bool = False) -> int:
        """A torch CUDA tensor is copied on the context's stream at the call (after the
        work torch's current stream has queued so far), or with zero_copy=True read in place
        by the commit that consumes it: the tensor is then kept referenced here until
        stats() shows no pending put (include/mel.h reservoir_put, field_on_device 2)."""
        Xa = np.ascontiguousarray(X, dtype=np.float32)
        if hasattr(field, "data_ptr"):                       # torch tensor
            on_dev = (2 if zero_copy else 1) if field.is_cuda else 0
            ptr = C.c_void_p(field.data_ptr())
            if field.is_cuda:
                import torch
                cur = torch.cuda.current_stream(field.device)
                if cur.cuda_stream != getattr(self, "_stream", None):
                    ev = torch.cuda.Event()
                    ev.record(cur)
                    self._check(self.lib.mel_stream_wait_event(self.h, C.c_void_p(ev.cuda_event)))
                if zero_copy:
                    if not hasattr(self, "_zc_refs"):
                        self._zc_refs = []
                    self._zc_refs.append(field)
        else:
            field = np.ascontiguousarray(field, dtype=np.float32)
            on_dev, ptr = 0, field.ctypes.data_as(C.c_void_p)
        return self._check(self.lib.reservoir_put(self.h, sim, t, _fptr(Xa), ptr, on_dev), (OK, EAGAIN))

    def close(self) -> int:
        return self._check(self.lib.reservoir_close(self.h))

    def copy_params_from(self, src: "Context"):
        """mel_params_copy(self, src): src's parameters into this context (another GPU),
        asynchronous on both streams."""
        st = self.lib.mel_params_copy(self.h, src.h)
        if st != OK:
            raise MelError(st, self.lib.mel_last_error(src.h).decode(errors="replace"))

    def put_generated(self, gen: "Heat", sims, X, t):
        """reservoir_put_generated: fields made on this GPU by the heat client; returns
        (status, n_put)."""
        sims = np.ascontiguousarray(sims, np.uint32)
        Xa = np.ascontiguousarray(X, np.float32).reshape(-1, 5)
        ta = np.ascontiguousarray(t, np.uint32)
        n = C.c_uint32(0)
        st = self._check(self.lib.reservoir_put_generated(self.h, gen.h, _u32p(sims), _f32p(Xa), _u32p(ta), len(ta),
                                                          C.byref(n)), (OK, EAGAIN))
        return st, n.value

    def train_offline(self, ds: "Dataset", seed: int, epoch: int, first_batch: int = 0, n_batches: int = 1 << 30,
                      want_losses: bool = True):
        """surrogate_train_offline: returns (steps, losses or None)."""
        nb = max(0, min(n_batches, ds.count // self.cfg.batch - first_batch))
        losses = np.zeros(max(nb, 1), np.float64) if want_losses else None
        steps = C.c_uint32(0)
        self._check(self.lib.surrogate_train_offline(
            self.h, ds.h, seed, epoch, first_batch, n_batches,
            losses.ctypes.data_as(C.POINTER(C.c_double)) if want_losses else None, C.byref(steps)))
        return steps.value, (losses[:steps.value] if want_losses else None)

    def ingest(self, ing: "Ingest", max_msgs: int = 1 << 30, timeout_us: int = 0):
        """reservoir_ingest: put up to max_msgs first-copy messages of an ingest ring.
        Returns (status, n_put); status OK or EOS."""
        n = C.c_uint32(0)
        st = self._check(self.lib.reservoir_ingest(self.h, ing.h, max_msgs, timeout_us, C.byref(n)), (OK, EOS))
        return st, n.value

    def sample(self, want_slots: bool = False, want_n: bool = False):
        """Returns (status, slots or None, n or None)."""
        slots = np.zeros(self.cfg.batch, dtype=np.int32) if want_slots else None
        n = C.c_uint32()
        r = self.lib.reservoir_sample_batch(self.h, slots.ctypes.data_as(C.POINTER(C.c_int32)) if want_slots else None,
                                            C.byref(n) if (want_slots or want_n) else None)
        self._check(r, (OK, EAGAIN))
        nn = n.value if (want_slots or want_n) else None
        return r, (slots[:nn] if want_slots else None), nn

    def step(self, want_loss: bool = True):
        loss = C.c_double()
        r = self.lib.surrogate_step(self.h, C.byref(loss) if want_loss else None)
        self.step_calls = getattr(self, "step_calls", 0) + 1
        self._check(r, (OK, EAGAIN, EOS))
        return r, (loss.value if (want_loss and r == OK) else None)

    def step_result(self, call: int):
        """(status, loss) of the call-th step() (0-based, one of the last 16), waiting
        only for that step's kernels."""
        loss, st = C.c_double(), C.c_int()
        self._check(self.lib.surrogate_step_result(self.h, call, C.byref(loss), C.byref(st)))
        return st.value, loss.value

    def eval(self, X, t, fields=None, want_pred=False):
        X = np.ascontiguousarray(X, dtype=np.float32)
        t = np.ascontiguousarray(t, dtype=np.uint32)
        n = X.shape[0]
        if fields is not None and hasattr(fields, "data_ptr"):      # torch tensor (device or host)
            fields = fields.float().contiguous()
            fptr = C.cast(C.c_void_p(fields.data_ptr()), C.POINTER(C.c_float))
            f = None
        else:
            f = np.ascontiguousarray(fields, dtype=np.float32) if fields is not None else None
            fptr = _fptr(f) if f is not None else None
        pred = np.zeros((n, self.cfg.n_field), dtype=np.float32) if want_pred else None
        mse = C.c_double()
        self._check(self.lib.surrogate_eval(self.h, _fptr(X), t.ctypes.data_as(C.POINTER(C.c_uint32)),
                                            fptr, n, C.byref(mse),
                                            _fptr(pred) if want_pred else None))
        return mse.value, pred

    def stats(self) -> dict:
        s = _Stats()
        self._check(self.lib.reservoir_stats(self.h, C.byref(s)))
        d = {k: getattr(s, k) for k, _ in _Stats._fields_ if k != "hist"}
        d["hist"] = np.array(list(s.hist), dtype=np.int64)
        if d.get("pending", 1) == 0:
            self._zc_refs = []                    # every zero-copy put has been committed
        return d

    def save_reservoir(self) -> np.ndarray:
        """The buffer's checkpoint blob (include/mel.h reservoir_save)."""
        n = C.c_uint64()
        self._check(self.lib.reservoir_checkpoint_bytes(self.h, C.byref(n)))
        blob = np.empty(n.value, dtype=np.uint8)
        self._check(self.lib.reservoir_save(self.h, blob.ctypes.data_as(C.c_void_p)))
        return blob

    def load_reservoir(self, blob: np.ndarray):
        blob = np.ascontiguousarray(blob, dtype=np.uint8)
        self._check(self.lib.reservoir_load(self.h, blob.ctypes.data_as(C.c_void_p)))

    def dump(self, payload: bool = True) -> dict:
        Cn, N = self.cfg.capacity, self.cfg.n_field
        sim = np.zeros(Cn, np.uint32); t = np.zeros(Cn, np.uint32); X = np.zeros((Cn, 5), np.float32)
        seen = np.zeros(Cn, np.uint32); ps = np.zeros(Cn, np.uint64)
        pl = None
        if payload:
            pl = np.zeros((Cn, N), np.float32 if self.cfg.storage == STORE_F32 else np.uint16)
        v = lambda a: a.ctypes.data_as(C.c_void_p)
        self._check(self.lib.reservoir_dump(self.h, v(sim), v(t), v(X), v(seen), v(ps), v(pl) if payload else None))
        return dict(sim=sim, t=t, X=X, seen=seen, put_seq=ps, payload=pl)

    # -- parameters / state ------------------------------------------------------------
    def _arrays(self):
        return [np.zeros(s, dtype=np.float32) if s[1] != 1 else np.zeros(s[0], dtype=np.float32)
                for s in self.shapes]

    @staticmethod
    def _ptrs(arrs):
        return (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])

    def get_params(self):
        out = self._arrays()
        self._check(self.lib.mel_get_params(self.h, self._ptrs(out)))
        return out

    def set_params(self, tensors):
        arrs = [np.ascontiguousarray(t, dtype=np.float32) for t in tensors]
        self._check(self.lib.mel_set_params(self.h, self._ptrs(arrs)))

    def get_state(self):
        p, m, v = self._arrays(), self._arrays(), self._arrays()
        sv = _StateView()
        pp, mp, vp = self._ptrs(p), self._ptrs(m), self._ptrs(v)
        sv.p, sv.m, sv.v = C.cast(pp, C.POINTER(C.c_void_p)), C.cast(mp, C.POINTER(C.c_void_p)), C.cast(vp, C.POINTER(C.c_void_p))
        self._check(self.lib.mel_get_state(self.h, C.byref(sv)))
        return dict(p=p, m=m, v=v, k=sv.adam_step, S=sv.samples_seen)

    def set_state(self, st):
        p = [np.ascontiguousarray(x, np.float32) for x in st["p"]]
        m = [np.ascontiguousarray(x, np.float32) for x in st["m"]]
        v = [np.ascontiguousarray(x, np.float32) for x in st["v"]]
        sv = _StateView()
        pp, mp, vp = self._ptrs(p), self._ptrs(m), self._ptrs(v)
        sv.p, sv.m, sv.v = C.cast(pp, C.POINTER(C.c_void_p)), C.cast(mp, C.POINTER(C.c_void_p)), C.cast(vp, C.POINTER(C.c_void_p))
        sv.adam_step, sv.samples_seen = st["k"], st["S"]
        self._check(self.lib.mel_set_state(self.h, C.byref(sv)))

    # -- misc ---------------------------------------------------------------------------
    def sync(self):
        self._check(self.lib.mel_sync(self.h))

    def kernel_time(self, k: int):
        ms, n = C.c_double(), C.c_uint64()
        self._check(self.lib.mel_kernel_time(self.h, k, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    def kernel_time_reset(self):
        self._check(self.lib.mel_kernel_time_reset(self.h))

    def debug_counters(self, n: int = 160 * 32 + 64 * 12 + 17 * 8):
        out = np.zeros(n, dtype=np.uint64)
        self._check(self.lib.mel_debug_counters(self.h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n))
        return out

    def set_flags(self, flags: int):
        self._check(self.lib.mel_set_flags(self.h, flags))

    def launch_count(self) -> int:
        n = C.c_uint64()
        self._check(self.lib.mel_launch_count(self.h, C.byref(n)))
        return n.value


class VirtualGroup:
    """`world` virtual ranks on one device (include/mel.h mel_create_virtual): .ctx[r] is
    rank r's Context (puts, samples, state, stats as usual); step() is the collective
    surrogate_step_virtual."""

    def __init__(self, cfg: Config, world: int, device: int = 0, stream: int | None = None):
        self.lib = load_library()
        self.cfg, self.world = cfg, world
        self._c = cfg.to_c()
        hs = (C.c_void_p * world)()
        r = self.lib.mel_create_virtual(C.byref(self._c), world, device, C.c_void_p(stream) if stream else None, hs)
        if r != OK:
            raise MelError(r, "mel_create_virtual failed (see stderr)")
        self._hs = hs
        self.ctx = [Context._from_handle(cfg, C.c_void_p(hs[q]), self.lib) for q in range(world)]
        self.step_calls = 0

    def step(self, want_loss: bool = True):
        loss = C.c_double()
        r = self.lib.surrogate_step_virtual(self._hs, self.world, C.byref(loss) if want_loss else None)
        self.step_calls += 1
        self.ctx[0]._check(r, (OK, EAGAIN, EOS))
        return r, (loss.value if (want_loss and r == OK) else None)

    def close(self):
        for c in getattr(self, "ctx", []):
            c.close_ctx()
        self.ctx = []

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Ingest:
    """Server side of one rank's ingest ring (include/mel_ingest.h)."""

    def __init__(self, name: str, rank: int, n_field: int, slots: int, expected_clients: int = 0, lib=None):
        self.lib = lib or load_library()
        self.h = C.c_void_p()
        st = self.lib.mel_ingest_create(name.encode(), rank, n_field, slots, expected_clients, C.byref(self.h))
        if st != OK:
            raise MelError(st, "mel_ingest_create(%s, %d)" % (name, rank))
        self.n_field = n_field

    def next(self, timeout_us: int = 0):
        """(status, msg) with msg = dict(sim_id, t, X, field (a copy), ticket) when status == OK."""
        m = _IngestMsg()
        st = self.lib.mel_ingest_next(self.h, C.byref(m), timeout_us)
        if st < 0:
            raise MelError(st, "mel_ingest_next")
        if st != OK:
            return st, None
        field = np.ctypeslib.as_array(m.field, shape=(self.n_field,)).copy()
        return st, dict(sim_id=m.sim_id, t=m.t, X=np.array(m.X[:], dtype=np.float32), field=field, ticket=m.ticket)

    def release(self):
        st = self.lib.mel_ingest_release(self.h)
        if st != OK:
            raise MelError(st, "mel_ingest_release")

    def outstanding(self) -> int:
        return int(self.lib.mel_ingest_outstanding(self.h))

    def stats(self) -> dict:
        s = _IngestStats()
        self.lib.mel_ingest_stats_get(self.h, C.byref(s))
        return {k: int(getattr(s, k)) for k, _ in _IngestStats._fields_}

    def destroy(self):
        if self.h:
            self.lib.mel_ingest_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


class Client:
    """A simulation client: init_communication / send / finalize_communication."""

    def __init__(self, name: str, world: int, client_id: int, lib=None):
        self.lib = lib or load_ingest_library()
        self.h = C.c_void_p()
        st = self.lib.mel_client_open(name.encode(), world, client_id, C.byref(self.h))
        if st != OK:
            raise MelError(st, "mel_client_open(%s)" % name)

    def send(self, t: int, X, field_f64, timeout_us: int = 10_000_000) -> int:
        Xa = np.ascontiguousarray(X, dtype=np.float32)
        f = np.ascontiguousarray(field_f64, dtype=np.float64)
        st = self.lib.mel_client_send(self.h, t, Xa.ctypes.data_as(C.POINTER(C.c_float)),
                                      f.ctypes.data_as(C.POINTER(C.c_double)), timeout_us)
        if st < 0:
            raise MelError(st, "mel_client_send")
        return st

    def finalize(self, timeout_us: int = 10_000_000) -> int:
        st = self.lib.mel_client_finalize(self.h, timeout_us)
        if st < 0:
            raise MelError(st, "mel_client_finalize")
        return st

    def close(self):
        if self.h:
            self.lib.mel_client_close(self.h)
            self.h = C.c_void_p()


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _f32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def write_dataset(path: str, n_field: int, records) -> int:
    """mel_dataset_create/append/finish over an iterable of (sim, t, X[5], field fp32)."""
    lib = load_library()
    w = C.c_void_p()
    st = lib.mel_dataset_create(path.encode(), n_field, C.byref(w))
    if st != OK:
        raise MelError(st, "mel_dataset_create(%s)" % path)
    n = 0
    for sim, t, X, f in records:
        Xa = np.ascontiguousarray(X, np.float32)
        fa = np.ascontiguousarray(f, np.float32)
        st = lib.mel_dataset_append(w, sim, t, _f32p(Xa), _f32p(fa))
        if st != OK:
            lib.mel_dataset_finish(w)
            raise MelError(st, "mel_dataset_append")
        n += 1
    st = lib.mel_dataset_finish(w)
    if st != OK:
        raise MelError(st, "mel_dataset_finish")
    return n


def epoch_order(count: int, seed: int, epoch: int) -> np.ndarray:
    perm = np.zeros(count, np.uint32)
    st = load_library().mel_dataset_epoch_order(count, seed, epoch, _u32p(perm))
    if st != OK:
        raise MelError(st, "mel_dataset_epoch_order")
    return perm


class Dataset:
    """Reader of a file dataset (include/mel_dataset.h) with `threads` loader workers."""

    def __init__(self, path: str, threads: int = 8):
        self.lib = load_library()
        self.h = C.c_void_p()
        st = self.lib.mel_dataset_open(path.encode(), threads, C.byref(self.h))
        if st != OK:
            raise MelError(st, "mel_dataset_open(%s)" % path)
        self.count = int(self.lib.mel_dataset_count(self.h))
        self.n_field = int(self.lib.mel_dataset_n_field(self.h))

    def read(self, idx, fields: bool = True):
        idx = np.ascontiguousarray(idx, np.uint32)
        n = len(idx)
        sim = np.zeros(n, np.uint32); t = np.zeros(n, np.uint32); X = np.zeros((n, 5), np.float32)
        F = np.zeros((n, self.n_field), np.float32) if fields else None
        st = self.lib.mel_dataset_read(self.h, _u32p(idx), n, _u32p(sim), _u32p(t), _f32p(X),
                                       _f32p(F) if fields else None, self.n_field)
        if st != OK:
            raise MelError(st, "mel_dataset_read")
        return sim, t, X, F

    def close(self):
        if self.h:
            self.lib.mel_dataset_close(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Heat:
    """The on-device heat-equation client (include/mel_heat.h): builds the fp64 basis on
    the current GPU; fields(X, t) -> fp32 device fields (torch tensors)."""

    def __init__(self, n: int, tau: int, alpha: float = 1.0, dt: float = 0.01, length: float = 1.0):
        self.lib = load_library()
        self.h = C.c_void_p()
        st = self.lib.mel_heat_create(n, tau, alpha, dt, length, C.byref(self.h))
        if st != OK:
            raise MelError(st, "mel_heat_create(%d, %d)" % (n, tau))
        self.n, self.tau = n, tau
        self.basis_bytes = int(self.lib.mel_heat_basis_bytes(self.h))

    def fields(self, X, t, stream=None):
        import torch
        X = torch.as_tensor(X, dtype=torch.float32, device="cuda").reshape(-1, 5).contiguous()
        t = torch.as_tensor(t, dtype=torch.int32, device="cuda").contiguous()
        out = torch.empty((X.shape[0], self.n * self.n), dtype=torch.float32, device="cuda")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        st = self.lib.mel_heat_fields(self.h, C.c_void_p(X.data_ptr()), C.c_void_p(t.data_ptr()), X.shape[0],
                                      C.c_void_p(out.data_ptr()), C.c_void_p(s))
        if st != OK:
            raise MelError(st, "mel_heat_fields")
        return out

    def destroy(self):
        if self.h:
            self.lib.mel_heat_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
