"""Python mirror of the reference's md_hom operator interface over the B200
C ABI (include/mdh_b200.h, libmdh_b200.so).

The names follow the reference so the parity tests read like its own tests:

    reference (C++, proj/include/mdh/)           here
    -------------------------------------------  ------------------------------------
    parse_computation_json (json_io.hpp:15)      Plan(spec, ...) takes the same JSON
    reference_execute(e, inputs) (highlevel:62)  execute(spec, inputs)     -> outputs
    interpret(lower(e, m, cfg), e, inputs)       execute(spec, inputs, asm=m, config=cfg)
    compiled_time_objective(e, m, cfg)           b200_time_objective(spec, asm, cfg)
    tune(e, m, cs, budget, obj, seed)            tune(spec, asm, budget, seed)
    validate(cfg, e, m, cs)                      validate_config(spec, asm, cfg)

Device memory, streams and the torch.distributed plumbing come from PyTorch;
all computation happens in the CUDA kernels of libmdh_b200.so.  There is no
CPU fallback: if the library or a GPU is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import json
import os
from typing import Any, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MDHB_LIB") or os.path.join(_HERE, "libmdh_b200.so")  # MDHB_LIB: variant builds (dev aid)

F32, F64, I32, I64 = 0, 1, 2, 3
MATH_FFMA, MATH_TF32, MATH_BF16 = 0, 1, 2
_NP = {F32: np.float32, F64: np.float64, I32: np.int32, I64: np.int64}

EXPORTED = [
    "mdh_b200_default_options", "mdh_b200_plan_create", "mdh_b200_plan_destroy", "mdh_b200_buffer_count",
    "mdh_b200_buffer_info", "mdh_b200_run", "mdh_b200_run_host", "mdh_b200_time", "mdh_b200_describe",
    "mdh_b200_validate_config", "mdh_b200_tune", "mdh_b200_tune_ex", "mdh_b200_simcost", "mdh_b200_lowered",
    "mdh_b200_launches_per_run", "mdh_b200_register_combine", "mdh_b200_combine_info",
    "mdh_b200_mplan_create", "mdh_b200_mplan_destroy", "mdh_b200_mplan_describe", "mdh_b200_mplan_shard_buffer",
    "mdh_b200_mplan_shard_plan", "mdh_b200_mplan_run", "mdh_b200_mplan_run_host", "mdh_b200_mplan_iterate",
    "mdh_b200_mplan_time", "mdh_b200_nccl_unique_id", "mdh_b200_rank_plan_create", "mdh_b200_time_synthetic", "mdh_b200_tune_space", "mdh_b200_shard_spec",
    "mdh_b200_kernel_source", "mdh_b200_last_error", "mdh_b200_version",
]
OBJ_TIME, OBJ_SIMCOST = 0, 1


class MdhError(RuntimeError):
    """Failure with the reference's stable error code (error.hpp:9-17)."""

    def __init__(self, msg: str):
        super().__init__(msg)
        self.code = msg.split(":", 1)[0]


class Options(ctypes.Structure):
    _fields_ = [("float_storage", ctypes.c_int), ("int_storage", ctypes.c_int), ("math", ctypes.c_int),
                ("device", ctypes.c_int), ("family", ctypes.c_int), ("split_dim", ctypes.c_int)]


_lib = None


def lib():
    """Loads libmdh_b200.so -- raises if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MdhError(f"LibraryMissing: {LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.mdh_b200_last_error.restype = ctypes.c_char_p
        L.mdh_b200_version.restype = ctypes.c_char_p
        c, v, i64, d = ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)
        L.mdh_b200_simcost.argtypes = [c, c, c, d, c, i64, ctypes.POINTER(ctypes.c_int64)]
        L.mdh_b200_lowered.argtypes = [c, c, c, c, i64, ctypes.POINTER(ctypes.c_int64)]
        L.mdh_b200_tune_ex.argtypes = [c, c, v, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, c, c, i64, c,
                                       i64, d]
        L.mdh_b200_tune.argtypes = [c, c, v, ctypes.c_int, ctypes.c_uint64, c, i64, c, i64, d]
        _lib = L
    return _lib


def _check(rc):
    if rc:
        raise MdhError(lib().mdh_b200_last_error().decode())


def _text(spec) -> bytes:
    if isinstance(spec, (dict, list)):
        spec = json.dumps(spec)
    return spec.encode() if isinstance(spec, str) else spec


def options(float_storage=F32, int_storage=I64, math=MATH_FFMA, device=0, generic=False, split_dim=0) -> Options:
    o = Options()
    lib().mdh_b200_default_options(ctypes.byref(o))
    o.float_storage, o.int_storage, o.math, o.device, o.family = float_storage, int_storage, math, device, int(generic)
    o.split_dim = split_dim
    return o


def _ptr_array(ptrs):
    return (ctypes.c_void_p * max(1, len(ptrs)))(*ptrs)


class Plan:
    """An md_hom bound to an instantiated sm_100a kernel template."""

    def __init__(self, spec, asm: str = "B200", config=None, float_storage=F32, int_storage=I64,
                 math=MATH_FFMA, device=0, generic=False, _handle=None):
        self.spec = spec if isinstance(spec, str) else json.dumps(spec)
        self._h = ctypes.c_void_p()
        self.opts = options(float_storage, int_storage, math, device, generic)
        if _handle is not None:  # built by another constructor (rank plans)
            self._h = _handle
        else:
            cfg = None if config is None else _text(config)
            _check(lib().mdh_b200_plan_create(_text(self.spec), _text(asm), cfg, ctypes.byref(self.opts),
                                              ctypes.byref(self._h)))
        self.device = device
        self.inputs = [self.buffer_info(0, b) for b in range(self._count(0))]
        self.outputs = [self.buffer_info(1, b) for b in range(self._count(1))]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mdh_b200_plan_destroy(h)
            self._h = ctypes.c_void_p()

    close = __del__

    def _count(self, side):
        n = ctypes.c_int()
        _check(lib().mdh_b200_buffer_count(self._h, side, ctypes.byref(n)))
        return n.value

    def buffer_info(self, side, b):
        dims = (ctypes.c_int64 * 16)()
        rank, dt, nb = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(lib().mdh_b200_buffer_info(self._h, side, b, dims, ctypes.byref(rank), ctypes.byref(dt),
                                          ctypes.byref(nb)))
        return {"shape": tuple(dims[r] for r in range(rank.value)), "dtype": dt.value, "bytes": nb.value,
                "np": _NP[dt.value]}

    def describe(self) -> dict:
        need = ctypes.c_int64()
        _check(lib().mdh_b200_describe(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(lib().mdh_b200_describe(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def kernel_source(self) -> str:
        """CUDA source of the NVRTC-compiled kernel (emitted family), else ""."""
        need = ctypes.c_int64()
        _check(lib().mdh_b200_kernel_source(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(max(1, need.value))
        _check(lib().mdh_b200_kernel_source(self._h, buf, need.value, ctypes.byref(need)))
        return buf.value.decode()

    @property
    def launches(self) -> int:
        n = ctypes.c_int()
        _check(lib().mdh_b200_launches_per_run(self._h, ctypes.byref(n)))
        return n.value

    # ---- device-resident (torch tensors as plumbing) --------------------
    def empty(self, side, device=None):
        import torch
        tdt = {F32: torch.float32, F64: torch.float64, I32: torch.int32, I64: torch.int64}
        infos = self.inputs if side == 0 else self.outputs
        dev = device or f"cuda:{self.device}"
        return [torch.empty(i["shape"], dtype=tdt[i["dtype"]], device=dev) for i in infos]

    def _dev_ptrs(self, tensors, infos):
        ptrs = []
        for t, i in zip(tensors, infos):
            if not t.is_cuda or not t.is_contiguous():
                raise MdhError("InvalidArgument: device buffers must be contiguous CUDA tensors")
            if tuple(t.shape) != i["shape"] or t.element_size() * t.numel() != i["bytes"]:
                raise MdhError(f"BufferTooSmall: expected shape {i['shape']} / {i['bytes']} bytes")
            ptrs.append(t.data_ptr())
        return _ptr_array(ptrs)

    def run(self, d_in, d_out, stream=None):
        """mdh_kernel(in..., out...) on device buffers, async on `stream`."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        _check(lib().mdh_b200_run(self._h, self._dev_ptrs(d_in, self.inputs), self._dev_ptrs(d_out, self.outputs),
                                  ctypes.c_void_p(stream)))

    def time(self, d_in, d_out, warmup=3, reps=5, flush_l2=True):
        """(median seconds per run, median seconds of the dominant kernel)."""
        med, ker = ctypes.c_double(), ctypes.c_double()
        _check(lib().mdh_b200_time(self._h, self._dev_ptrs(d_in, self.inputs), self._dev_ptrs(d_out, self.outputs),
                                   warmup, reps, int(flush_l2), ctypes.byref(med), ctypes.byref(ker)))
        return med.value, ker.value

    # ---- host buffers (the end-to-end path) ------------------------------
    def run_host(self, h_in: Sequence[np.ndarray], h_out: Optional[List[np.ndarray]] = None):
        ins = []
        for x, i in zip(h_in, self.inputs):
            a = np.ascontiguousarray(x, dtype=i["np"])
            if a.shape != i["shape"]:
                raise MdhError(f"BufferTooSmall: input shape {a.shape} != {i['shape']}")
            ins.append(a)
        if h_out is None:
            h_out = [np.empty(i["shape"], dtype=i["np"]) for i in self.outputs]
        _check(lib().mdh_b200_run_host(self._h, _ptr_array([a.ctypes.data for a in ins]),
                                       _ptr_array([a.ctypes.data for a in h_out]), None))
        return h_out


# ---------------------------------------------------------------- DEV layer
def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (128 bytes) -- made on one rank, broadcast by the caller."""
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().mdh_b200_nccl_unique_id(buf))
    return bytes(buf)


def shard_spec(spec, world, rank, split_dim=0, asm="MultiB200", config=None) -> dict:
    """Host only: the DEV layer's shard `rank` of `world` (the C++ split rule
    of mdh_b200_rank_plan_create) -> {"computation", "config", "shard"}."""
    need = ctypes.c_int64()
    args = (_text(spec), _text(asm), None if config is None else _text(config), int(world), int(rank), int(split_dim))
    _check(lib().mdh_b200_shard_spec(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_shard_spec(*args, buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def rank_plan(spec, world, rank, device=0, nccl_id: Optional[bytes] = None, asm="MultiB200", config=None,
              split_dim=0, **kw) -> Plan:
    """One process per GPU: rank `rank`'s shard of the md_hom split over the
    GPU layer (mdh_b200_rank_plan_create).  With `nccl_id` a point-wise split
    all-reduces its outputs over NCCL inside run(); without, the caller
    combines (describe()["template"]["shard"] says how)."""
    o = options(device=device, split_dim=split_dim, **kw)
    h = ctypes.c_void_p()
    idb = None if nccl_id is None else (ctypes.c_ubyte * 128)(*nccl_id)
    text = spec if isinstance(spec, str) else json.dumps(spec)
    _check(lib().mdh_b200_rank_plan_create(_text(text), _text(asm), None if config is None else _text(config),
                                           ctypes.byref(o), int(world), int(rank), idb, ctypes.byref(h)))
    p = Plan(text, device=device, _handle=h)
    p.opts = o
    return p


class MultiPlan:
    """mdh_b200_mplan_*: one process drives G shards of the md_hom (device_ids
    may repeat -- shards then share a device and combine through the peer
    kernel)."""

    def __init__(self, spec, n_gpus, device_ids=None, asm="MultiB200", config=None, split_dim=0, **kw):
        self.spec = spec if isinstance(spec, str) else json.dumps(spec)
        self.G = int(n_gpus)
        self.devices = list(device_ids) if device_ids is not None else list(range(self.G))
        o = options(split_dim=split_dim, **kw)
        self._h = ctypes.c_void_p()
        devs = (ctypes.c_int * self.G)(*self.devices)
        _check(lib().mdh_b200_mplan_create(_text(self.spec), _text(asm), None if config is None else _text(config),
                                           ctypes.byref(o), self.G, devs, ctypes.byref(self._h)))
        n_in, n_out = len(json.loads(self.spec)["inputs"]), len(json.loads(self.spec)["outputs"])
        self.inputs = [[self.shard_buffer(g, 0, b) for b in range(n_in)] for g in range(self.G)]
        self.outputs = [[self.shard_buffer(g, 1, b) for b in range(n_out)] for g in range(self.G)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.mdh_b200_mplan_destroy(h)
            self._h = ctypes.c_void_p()

    def describe(self) -> dict:
        need = ctypes.c_int64()
        _check(lib().mdh_b200_mplan_describe(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(need.value)
        _check(lib().mdh_b200_mplan_describe(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def shard_buffer(self, g, side, b):
        dims = (ctypes.c_int64 * 16)()
        sr, st, rank, dt, nb = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(lib().mdh_b200_mplan_shard_buffer(self._h, g, side, b, ctypes.byref(sr), ctypes.byref(st), dims,
                                                 ctypes.byref(rank), ctypes.byref(dt), ctypes.byref(nb)))
        return {"slab_rank": sr.value, "start": st.value, "shape": tuple(dims[r] for r in range(rank.value)),
                "dtype": dt.value, "bytes": nb.value, "np": _NP[dt.value]}

    def empty(self, side):
        import torch
        tdt = {F32: torch.float32, F64: torch.float64, I32: torch.int32, I64: torch.int64}
        infos = self.inputs if side == 0 else self.outputs
        return [[torch.empty(i["shape"], dtype=tdt[i["dtype"]], device=f"cuda:{self.devices[g]}") for i in infos[g]]
                for g in range(self.G)]

    def slab(self, g, side, b, array):
        """Shard g's slab of a GLOBAL buffer (numpy or torch)."""
        i = (self.inputs if side == 0 else self.outputs)[g][b]
        if i["slab_rank"] < 0:
            return array
        idx = [slice(None)] * array.ndim
        r = i["slab_rank"]
        idx[r] = slice(i["start"], i["start"] + i["shape"][r])
        return array[tuple(idx)]

    def _pp(self, bufs):
        rows = [_ptr_array([t.data_ptr() for t in row]) for row in bufs]
        arr = (ctypes.c_void_p * self.G)(*[ctypes.cast(r, ctypes.c_void_p) for r in rows])
        return arr, rows

    def run(self, d_in, d_out):
        a, ka = self._pp(d_in)
        b, kb = self._pp(d_out)
        _check(lib().mdh_b200_mplan_run(self._h, a, b, None))

    def iterate(self, d_v, d_w, sweeps):
        a, ka = self._pp(d_v)
        b, kb = self._pp(d_w)
        _check(lib().mdh_b200_mplan_iterate(self._h, a, b, int(sweeps), None))

    def time(self, d_in, d_out, warmup=2, reps=5):
        a, ka = self._pp(d_in)
        b, kb = self._pp(d_out)
        med = ctypes.c_double()
        _check(lib().mdh_b200_mplan_time(self._h, a, b, warmup, reps, ctypes.byref(med)))
        return med.value

    def run_host(self, h_in, h_out=None):
        """GLOBAL host buffers in, GLOBAL host outputs out (slabs scattered / gathered)."""
        spec = json.loads(self.spec)
        ins = [np.ascontiguousarray(x, dtype=i["np"]) for x, i in zip(h_in, self.inputs[0])]
        if h_out is None:
            h_out = []
            for b in range(len(spec["outputs"])):
                i = self.outputs[0][b]
                shp = list(i["shape"])
                if i["slab_rank"] >= 0:
                    shp[i["slab_rank"]] = max(self.outputs[g][b]["start"] + self.outputs[g][b]["shape"][i["slab_rank"]]
                                              for g in range(self.G))
                h_out.append(np.empty(shp, dtype=i["np"]))
        _check(lib().mdh_b200_mplan_run_host(self._h, _ptr_array([a.ctypes.data for a in ins]),
                                             _ptr_array([a.ctypes.data for a in h_out])))
        return h_out


def execute(spec, inputs: Sequence[np.ndarray], asm="B200", config=None, **kw) -> List[np.ndarray]:
    """reference_execute / interpret(lower(...)) on the B200: host in, host out."""
    return Plan(spec, asm, config, **kw).run_host(inputs)


def b200_time_objective(spec, asm="B200", config=None, reps=5, **kw) -> float:
    """compiled_time_objective's role (autotuner.hpp:73): median seconds of the
    instantiated kernel on synthetic device inputs, L2 flushed between reps."""
    import torch
    p = Plan(spec, asm, config, **kw)
    ins = p.empty(0)
    for t in ins:
        if t.is_floating_point():
            t.uniform_(-1, 1)
        else:
            t.random_(0, 3)
    outs = p.empty(1)
    # the fills ran on torch's stream; mdh_b200_time times on the plan's own
    # non-blocking stream, which does not order after them
    torch.cuda.synchronize()
    med, _ = p.time(ins, outs, warmup=1, reps=reps)
    return med


def validate_config(spec, asm, config) -> str:
    need = ctypes.c_int64()
    _check(lib().mdh_b200_validate_config(_text(spec), _text(asm), _text(config), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_validate_config(_text(spec), _text(asm), _text(config), buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def tune(spec, asm="B200", budget=20, seed=0, **kw):
    """mdh::tune with the on-device objective -> (best_config_json, history_csv, best_seconds)."""
    o = options(**kw)
    best = ctypes.create_string_buffer(1 << 20)
    hist = ctypes.create_string_buffer(1 << 20)
    secs = ctypes.c_double()
    _check(lib().mdh_b200_tune(_text(spec), _text(asm), ctypes.byref(o), budget, ctypes.c_uint64(seed), best,
                               1 << 20, hist, 1 << 20, ctypes.byref(secs)))
    return best.value.decode(), hist.value.decode(), secs.value


def tune_ex(spec, asm="B200", budget=20, seed=0, objective=OBJ_TIME, simcost_seeded=False, start_config=None, **kw):
    """mdh::tune with the objective choice (device time | SimCost), SimCost
    seeding of the random phase and an optional start configuration ->
    (best_config_json, history_csv, best_objective)."""
    o = options(**kw)
    best = ctypes.create_string_buffer(1 << 20)
    hist = ctypes.create_string_buffer(1 << 20)
    val = ctypes.c_double()
    _check(lib().mdh_b200_tune_ex(_text(spec), _text(asm), ctypes.byref(o), budget, ctypes.c_uint64(seed),
                                  int(objective), int(bool(simcost_seeded)), _text(start_config) if start_config else None,
                                  best, 1 << 20, hist, 1 << 20, ctypes.byref(val)))
    return best.value.decode(), hist.value.decode(), val.value


def tune_space(spec, family, asm="B200", **kw) -> list:
    """The tuner's enumerated candidates for a kernel family (host only)."""
    o = options(**kw)
    need = ctypes.c_int64()
    _check(lib().mdh_b200_tune_space(_text(spec), _text(asm), ctypes.byref(o), _text(family), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_tune_space(_text(spec), _text(asm), ctypes.byref(o), _text(family), buf, need.value,
                                     ctypes.byref(need)))
    return json.loads(buf.value.decode())


def simcost(spec, asm="B200", config=None):
    """mdh::simcost_objective (autotuner.cpp:58-62) -> (cost, trace totals dict).
    Host only: no GPU is touched."""
    cost = ctypes.c_double()
    need = ctypes.c_int64()
    cfg = _text(config) if config is not None else None
    _check(lib().mdh_b200_simcost(_text(spec), _text(asm), cfg, ctypes.byref(cost), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_simcost(_text(spec), _text(asm), cfg, ctypes.byref(cost), buf, need.value, ctypes.byref(need)))
    return cost.value, json.loads(buf.value.decode())


def lowered(spec, asm="B200", config=None) -> str:
    """mdh::lower(expr, model, cfg).pretty() (lowering.cpp:185-222). Host only."""
    need = ctypes.c_int64()
    cfg = _text(config) if config is not None else None
    _check(lib().mdh_b200_lowered(_text(spec), _text(asm), cfg, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_lowered(_text(spec), _text(asm), cfg, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def register_combine(name, arity, cuda_body, identity=(), assoc=True, comm=True, description=""):
    """Registers a custom combine operator usable as "pw:<name>" / "ps:<name>"
    (API extension; the reference's operator set is closed, mda.hpp:52).
    `cuda_body` folds the component tuple: statements over a0.. (accumulator
    lvalues) and b0.. (next value)."""
    _check(lib().mdh_b200_register_combine(_text(name), int(arity), _text(cuda_body),
                                           _text(",".join(identity)), int(bool(assoc)), int(bool(comm)),
                                           _text(description)))


def combine_info() -> list:
    need = ctypes.c_int64()
    _check(lib().mdh_b200_combine_info(None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().mdh_b200_combine_info(buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def version() -> str:
    return lib().mdh_b200_version().decode()
