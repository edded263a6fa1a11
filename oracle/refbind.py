"""TEST INFRASTRUCTURE -- ctypes binding of the UNMODIFIED reference library
(oracle/_ref/libmdh_ref.so, built by oracle/Makefile from /root/reference).

Used to pin the oracle restatement (tests/test_oracle.py), to generate the
golden vectors (tests/golden/make_golden.py) and as the CPU baseline
(bench.py --impl reference, cpu_baseline kind "reference").  Never on the
product path.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import subprocess
from typing import List, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(_HERE, "_ref", "libmdh_ref.so")
_lib = None


class RefError(Exception):
    def __init__(self, msg: str):
        super().__init__(msg)
        self.code = msg.split(":", 1)[0]


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError("RefUnavailable: oracle/_ref/libmdh_ref.so not built (make -C oracle ref)")
        _lib = ctypes.CDLL(REF_SO)
        _lib.ref_last_error.restype = ctypes.c_char_p
    return _lib


def _check(rc):
    if rc:
        raise RefError(lib().ref_last_error().decode())


def _b(s):
    return s.encode() if isinstance(s, str) else s


def buffer_info(comp_json: str, side: int, b: int):
    dims = (ctypes.c_int64 * 16)()
    rank, is_f = ctypes.c_int(), ctypes.c_int()
    _check(lib().ref_buffer_info(_b(comp_json), side, b, dims, ctypes.byref(rank), ctypes.byref(is_f)))
    return [dims[r] for r in range(rank.value)], bool(is_f.value)


def _n_bufs(comp_json, side):
    import json
    j = json.loads(comp_json)
    return len(j["inputs" if side == 0 else "outputs"])


def _prep(comp_json, inputs):
    ins = []
    for b, x in enumerate(inputs):
        _, is_f = buffer_info(comp_json, 0, b)
        ins.append(np.ascontiguousarray(x, dtype=np.float64 if is_f else np.int64))
    outs, defs = [], []
    for b in range(_n_bufs(comp_json, 1)):
        dims, is_f = buffer_info(comp_json, 1, b)
        outs.append(np.zeros(dims, dtype=np.float64 if is_f else np.int64))
        defs.append(np.zeros(dims, dtype=np.uint8))
    P = lambda arrs: (ctypes.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])  # noqa: E731
    return ins, outs, defs, P


def reference_execute(comp_json: str, inputs: Sequence[np.ndarray]):
    """mdh::reference_execute (highlevel.hpp:62-63) -> [(values, defined)]."""
    ins, outs, defs, P = _prep(comp_json, inputs)
    _check(lib().ref_execute(_b(comp_json), P(ins), P(outs), P(defs)))
    return [(o, d.astype(bool)) for o, d in zip(outs, defs)]


def interpret(comp_json: str, asm: str, cfg_json: str, inputs):
    """mdh::interpret(mdh::lower(...)) (interpreter.hpp:44-46)."""
    ins, outs, defs, P = _prep(comp_json, inputs)
    _check(lib().ref_interpret(_b(comp_json), _b(asm), _b(cfg_json or ""), P(ins), P(outs), P(defs)))
    return [(o, d.astype(bool)) for o, d in zip(outs, defs)]


def _string_call(fn, *args):
    need = ctypes.c_int64()
    _check(fn(*args, None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(fn(*args, buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def emit(comp_json: str, asm: str, cfg_json: str = "") -> str:
    """mdh::emit (codegen.hpp:38): the OpenMP C kernel `mdh_kernel`."""
    return _string_call(lib().ref_emit, _b(comp_json), _b(asm), _b(cfg_json))


def lowered(comp_json: str, asm: str, cfg_json: str = "") -> str:
    """mdh::lower(expr, model, cfg).pretty() (lowering.cpp:185-222)."""
    return _string_call(lib().ref_lowered, _b(comp_json), _b(asm), _b(cfg_json))


def sample_config(comp_json: str, asm: str, seed: int, reduced=True, model_rules=True) -> str:
    return _string_call(lib().ref_sample_config, _b(comp_json), _b(asm), ctypes.c_uint64(seed),
                        ctypes.c_int(int(reduced)), ctypes.c_int(int(model_rules)))


def validate(comp_json: str, asm: str, cfg_json: str, model_rules=True) -> str:
    """'' when valid, else '<rule>: <message>' of the first violation."""
    return _string_call(lib().ref_validate, _b(comp_json), _b(asm), _b(cfg_json), ctypes.c_int(int(model_rules)))


def simcost(comp_json: str, asm: str, cfg_json: str) -> float:
    v = ctypes.c_double()
    _check(lib().ref_simcost(_b(comp_json), _b(asm), _b(cfg_json), ctypes.byref(v)))
    return v.value


def fixture(name: str):
    comp = ctypes.create_string_buffer(1 << 16)
    cfg = ctypes.create_string_buffer(1 << 20)
    asm = ctypes.create_string_buffer(256)
    _check(lib().ref_fixture(_b(name), comp, 1 << 16, cfg, 1 << 20, asm, 256))
    return comp.value.decode(), cfg.value.decode(), asm.value.decode()


# ---- the reference's emitted OpenMP kernel as a CPU baseline ------------
class EmittedKernel:
    """Builds the kernel `emit` produces with the flags compile_and_run uses
    (emitted_runner.cpp:53-66: -O2 -fopenmp -ffp-contract=off), as a shared
    object, and calls `mdh_kernel(const T* in..., T* out...)` on numpy
    buffers.  The kernel source is the reference's; nothing is edited."""

    def __init__(self, comp_json: str, asm: str, cfg_json: str, cc: str = "/usr/bin/gcc"):
        self.comp_json = comp_json
        src = emit(comp_json, asm, cfg_json)
        key = hashlib.sha1(src.encode()).hexdigest()[:16]
        d = os.path.join(_HERE, "_ref", "emitted")
        os.makedirs(d, exist_ok=True)
        self.so = os.path.join(d, f"k_{key}.so")
        if not os.path.exists(self.so):
            cpath = os.path.join(d, f"k_{key}.c")
            with open(cpath, "w") as f:
                f.write(src)
            subprocess.check_call([cc, "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC",
                                   "-o", self.so, cpath])
        self.lib = ctypes.CDLL(self.so)

    def __call__(self, inputs: Sequence[np.ndarray], outputs: Sequence[np.ndarray]):
        args = [ctypes.c_void_p(a.ctypes.data) for a in list(inputs) + list(outputs)]
        self.lib.mdh_kernel(*args)
