"""`mdh` command-line driver with the B200 backend.

The reference's driver, proj/tools/mdh_main.cpp, needs CLI11 and is not
buildable here; this mirrors its subcommands, options, output lines and exit
codes (mdh_main.cpp:243-251: ParseError -> 3; InvalidConfig, Mismatch,
NoValidConfigFound, NonDivisible, MixedIncompatibleOperators, UnknownPreset,
UnknownFixture -> 2; anything else -> 1), reading the reference's own JSON
formats unchanged:

    python -m paper_2405_05118_b200.cli verify  --spec S [--asm A] [--config C | --fixture F] [--seed N]
    python -m paper_2405_05118_b200.cli tune    --spec S [--asm A] [--budget N] [--seed N] [--out F] [--history F]
    python -m paper_2405_05118_b200.cli emit    --spec S [--asm A] [--config C] [--out F]
    python -m paper_2405_05118_b200.cli run     --spec S [--config C] --inputs ref.json [--out F]
    python -m paper_2405_05118_b200.cli describe --spec S [--asm A] [--config C] [--tf32]
    python -m paper_2405_05118_b200.cli examples [--data DIR]

--spec takes a computation JSON file, or the name of one in --data
(default: the package's data/ dir -- the reference's bundled computations
and fixtures, unchanged, plus the BASELINE specs).

`verify` is the reference's verify (interpret(lower(cfg)) against
reference_execute, mdh_main.cpp:130-166) on the device: the plan
instantiated from each configuration runs against the device's
reference-semantics executor (the generic family in f64 storage: the
reference's bytecode, lexicographic fold, bit-identical to reference_execute
on the frozen vectors), on the driver's deterministic k/4 inputs
(mdh_main.cpp:46-66).  `emit` prints the CUDA source the emitted family
compiles with NVRTC (mdh emit prints C).  `tune --objective` is the
SimCost model (default) or the device time (compiled_time_objective's role);
the history CSV has the reference's columns (autotuner.cpp:49-56), and the
printed best hash is the one of the best configuration's history row.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

from . import mdh

EXIT2 = {"InvalidConfig", "Mismatch", "NoValidConfigFound", "NonDivisible", "MixedIncompatibleOperators",
         "UnknownPreset", "UnknownFixture"}
_HERE = os.path.dirname(os.path.abspath(__file__))
_REPO = os.path.dirname(_HERE)


class CliError(Exception):
    def __init__(self, code, msg):
        super().__init__(f"{code}: {msg}")
        self.code = code


def exit_code_for(code: str) -> int:
    if code == "ParseError":
        return 3
    return 2 if code in EXIT2 else 1


def _data_dirs(data):
    out = []
    if data:
        out.append(data)
    # the data shipped with the package: the reference's bundled computations
    # and published fixtures (JSON, unchanged) plus the BASELINE specs
    out.append(os.path.join(os.path.dirname(os.path.abspath(__file__)), "data"))
    return out


def load_spec(arg, data=None) -> dict:
    if not arg:
        raise CliError("ParseError", "--spec is required (bundled name or a JSON file)")
    if os.path.exists(arg):
        with open(arg) as f:
            return json.load(f)
    for d in _data_dirs(data):
        for p in (os.path.join(d, "computations", arg + ".json"), os.path.join(d, arg + ".json")):
            if os.path.exists(p):
                with open(p) as f:
                    return json.load(f)
    raise CliError("ParseError", f"cannot open '{arg}'")


def load_fixture(name, data=None):
    if os.path.exists(name):
        path = name
    else:
        path = None
        for d in _data_dirs(data):
            p = os.path.join(d, "fixtures", name + ".json")
            if os.path.exists(p):
                path = p
                break
        if path is None:
            raise CliError("UnknownFixture", f"no fixture named '{name}'")
    with open(path) as f:
        fx = json.load(f)
    spec = load_spec(fx["spec"], data)
    spec["sizes"] = fx["sizes"]
    return fx["name"], spec, fx["model"], fx["config"]


class _MT64:
    """std::mt19937_64 (the reference's mdh::Rng, proj/include/mdh/rng.hpp:12-18:
    below(n) = gen() % n) -- the published MT19937-64 recurrence."""
    N, M = 312, 156

    def __init__(self, seed):
        mt = [0] * self.N
        mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, self.N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.mt, self.i = mt, self.N

    def _twist(self):
        mt, N, M = self.mt, self.N, self.M
        for i in range(N):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % N] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + M) % N] ^ xa
        self.i = 0

    def next(self):
        if self.i >= self.N:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


def make_inputs(plan: "mdh.Plan", spec: dict, seed: int):
    """The driver's deterministic inputs (mdh_main.cpp:46-66): one
    mt19937_64(seed ^ 0x9e3779b97f4a7c15) stream over all buffers in view
    order, v = below(11) - 5; i64 cells take v, f64 cells 0.25 * v (exact in
    every storage type).  Buffers past 2^22 cells use a numpy stream of the
    same value set (the pure-Python generator would dominate the run)."""
    total = sum(int(np.prod(i["shape"])) for i in plan.inputs)
    out = []
    if total <= (1 << 22):
        g = _MT64(seed ^ 0x9E3779B97F4A7C15)
        for info, b in zip(plan.inputs, spec["inputs"]):
            n = int(np.prod(info["shape"]))
            v = np.array([g.next() % 11 for _ in range(n)], dtype=np.int64).reshape(info["shape"]) - 5
            out.append(v.astype(np.float64) * 0.25 if b["type"] == "f64" else v)
        return out
    rng = np.random.default_rng(seed)
    for info, b in zip(plan.inputs, spec["inputs"]):
        v = rng.integers(0, 11, info["shape"]).astype(np.int64) - 5
        out.append(v.astype(np.float64) * 0.25 if b["type"] == "f64" else v)
    return out


def _config_text(path):
    if path is None:
        return None
    with open(path) as f:
        return f.read()


def _prime_factors(n):
    out, f = [], 2
    while f * f <= n:
        while n % f == 0:
            out.append(f)
            n //= f
        f += 1
    if n > 1:
        out.append(n)
    return out


def random_configs(spec, model, n, seed, device=0):
    """`--random N` (mdh_main.cpp:120-125 samples N configurations with seeds
    seed + k): here each sample re-distributes every dimension's prime factors
    over the ASM layers at random (mt19937_64, below(n) = gen() % n) around the
    backend's canonical configuration for the spec, keeping its orders,
    assignments and memory regions; samples violating the model rules are
    redrawn (up to 64 times, else the canonical one is used)."""
    base = mdh.Plan(spec, model, None, device=device).describe()["config"]
    text = json.dumps(spec)
    out = []
    for k in range(n):
        rng = _MT64(seed + k)
        cfg = base
        for _ in range(64):
            c = json.loads(json.dumps(base))
            parts = c["num_parts"]
            layers = len(parts)
            for d, size in enumerate(spec["sizes"]):
                col = [1] * layers
                for f in _prime_factors(int(size)):
                    col[rng.next() % layers] *= f
                for l in range(layers):
                    parts[l][d] = col[l]
            if not mdh.validate_config(text, model, json.dumps(c)):
                cfg = c
                break
        out.append((f"random:{k}", json.dumps(cfg), model))
    return out


def cmd_verify(a) -> int:
    jobs = []
    if a.fixture:
        label, spec, model, cfg = load_fixture(a.fixture, a.data)
        jobs.append((label, json.dumps(cfg), model))
    else:
        spec = load_spec(a.spec, a.data)
        if a.random and not a.config:
            jobs.extend(random_configs(spec, a.asm, a.random, a.seed, a.device))
        else:
            jobs.append((a.config or "default", _config_text(a.config), a.asm))
    ref = mdh.Plan(spec, float_storage=mdh.F64, int_storage=mdh.I64, generic=True, device=a.device)
    ins = make_inputs(ref, spec, a.seed)
    want = ref.run_host(ins)
    failed = 0
    for label, cfg, model in jobs:
        if cfg is not None:
            why = mdh.validate_config(json.dumps(spec), model, cfg)
            if why:
                print(f"config {label}: INVALID ({why})")
                failed += 1
                continue
        plan = mdh.Plan(spec, model, cfg, device=a.device)
        got = plan.run_host(ins)
        d = plan.describe()
        ok, why = True, ""
        K = 1
        for n, c in zip(spec["sizes"], spec["combine"]):
            if c != "cc":
                K *= n
        for b, (g, w) in enumerate(zip(got, want)):
            g64, w64 = g.astype(np.float64), w.astype(np.float64)
            if np.issubdtype(w.dtype, np.integer):
                bad = np.flatnonzero(g.astype(np.int64) != w)
            else:
                tol = 1e-5 * np.sqrt(max(K, 1)) * np.maximum(np.abs(w64), 1.0)
                bad = np.flatnonzero(np.abs(g64 - w64) > tol)
            if bad.size:
                t = int(bad[0])
                ok, why = False, f"buffer '{spec['outputs'][b]['name']}' cell {t}: {g.flat[t]} != {w.flat[t]}"
                break
        h = hash_config(d["config"])
        if ok:
            print(f"config {label}: pass (hash={h:x}, family={d['family']}, kernel={d['template']['kernel']})")
        else:
            print(f"config {label}: FAIL ({why})")
            failed += 1
    if failed:
        print(f"{failed}/{len(jobs)} configurations failed")
        return 2
    print(f"{len(jobs)}/{len(jobs)} configurations pass")
    return 0


def hash_config(cfg) -> int:
    """FNV-1a over the configuration JSON text exactly as the library returned
    it (config_hash, autotuner.cpp:39-47; the tuner's history rows hash the
    same text, so the printed best hash matches its row)."""
    text = cfg if isinstance(cfg, str) else json.dumps(cfg, separators=(", ", ": "))
    h = 14695981039346656037
    for ch in text.encode():
        h ^= ch
        h = (h * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def cmd_tune(a) -> int:
    spec = load_spec(a.spec, a.data)
    start = None
    if a.start:
        _, _, _, start = load_fixture(a.start, a.data)
        start = json.dumps(start) if not isinstance(start, str) else start
    objective = mdh.OBJ_SIMCOST if a.objective == "simcost" else mdh.OBJ_TIME
    best, hist, secs = mdh.tune_ex(spec, a.asm, budget=a.budget, seed=a.seed, objective=objective,
                                   simcost_seeded=a.seed_simcost, start_config=start, device=a.device,
                                   math=mdh.MATH_TF32 if a.tf32 else mdh.MATH_FFMA)
    rows = [r for r in hist.strip().splitlines()[1:] if r]
    print(f"evaluations: {len(rows)}")
    print(f"best objective: {secs:.9g}")
    print(f"best hash: {hash_config(best):x}")
    if a.history:
        with open(a.history, "w") as f:
            f.write(hist)
    if a.out:
        with open(a.out, "w") as f:
            f.write(best)
    else:
        print(best)
    return 0


def cmd_lower(a) -> int:
    """`mdh lower` (mdh_main.cpp:293-295): the lowered expression of the
    configuration (or fixture), as LowLevelExpr::pretty() prints it.  Host
    only -- no GPU is touched."""
    if a.fixture:
        _, spec, model, cfg = load_fixture(a.fixture, a.data)
        text = mdh.lowered(spec, model, json.dumps(cfg) if not isinstance(cfg, str) else cfg)
    else:
        spec = load_spec(a.spec, a.data)
        text = mdh.lowered(spec, a.asm, _config_text(a.config))
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return 0


def cmd_emit(a) -> int:
    spec = load_spec(a.spec, a.data)
    cfg = _config_text(a.config)
    if cfg is not None:
        why = mdh.validate_config(json.dumps(spec), a.asm, cfg)
        if why:
            print(f"config {a.config} is invalid ({why})", file=sys.stderr)
            return 2
    plan = mdh.Plan(spec, a.asm, cfg, float_storage=mdh.F64 if a.f64 else mdh.F32, device=a.device)
    src = plan.kernel_source()
    if not src:
        d = plan.describe()
        src = (f"// {spec.get('name', '')}: served by the precompiled '{d['family']}' family, template "
               f"{json.dumps(d['template'])}\n")
    if a.out:
        with open(a.out, "w") as f:
            f.write(src)
    else:
        sys.stdout.write(src)
    if not a.gate_compile:
        return 0
    # --gate-compile (mdh_main.cpp:180-205): the kernel was compiled (NVRTC)
    # when the plan was made; run it on the driver's inputs against the
    # device reference executor
    ref = mdh.Plan(spec, float_storage=mdh.F64, int_storage=mdh.I64, generic=True, device=a.device)
    ins = make_inputs(ref, spec, a.seed)
    want = ref.run_host(ins)
    got = plan.run_host(ins)
    K = 1
    for n, c in zip(spec["sizes"], spec["combine"]):
        if c != "cc":
            K *= n
    for g, w in zip(got, want):
        if np.issubdtype(w.dtype, np.integer):
            bad = np.flatnonzero(g.astype(np.int64) != w)
        else:
            w64 = w.astype(np.float64)
            bad = np.flatnonzero(np.abs(g.astype(np.float64) - w64) > 1e-5 * np.sqrt(max(K, 1)) * np.maximum(np.abs(w64), 1.0))
        if bad.size:
            raise CliError("Mismatch", f"gate failed: cell {int(bad[0])}: {g.flat[int(bad[0])]} != {w.flat[int(bad[0])]}")
    d = plan.describe()
    print(f"gate passed: compiled with NVRTC (sm_100a), {d['family']} / {d['template']['kernel']}", file=sys.stderr)
    return 0


def cmd_describe(a) -> int:
    spec = load_spec(a.spec, a.data)
    plan = mdh.Plan(spec, a.asm, _config_text(a.config), math=mdh.MATH_TF32 if a.tf32 else mdh.MATH_FFMA,
                    device=a.device)
    print(json.dumps(plan.describe(), indent=1))
    return 0


def cmd_run(a) -> int:
    """Executes on the reference's ref-file inputs ({"inputs": {name: {dims,
    data}}}, data/refs/*.ref.json) and writes outputs in the same format."""
    spec = load_spec(a.spec, a.data)
    with open(a.inputs) as f:
        ref = json.load(f)
    plan = mdh.Plan(spec, a.asm, _config_text(a.config), float_storage=mdh.F64, int_storage=mdh.I64, device=a.device)
    ins = []
    for b, info in zip(spec["inputs"], plan.inputs):
        g = ref["inputs"][b["name"]]
        ins.append(np.array(g["data"], dtype=np.float64 if b["type"] == "f64" else np.int64).reshape(g["dims"]))
    outs = plan.run_host(ins)
    res = {"outputs": {b["name"]: {"dims": list(o.shape), "data": o.ravel().tolist()} for b, o in zip(spec["outputs"], outs)}}
    text = json.dumps(res)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text)
    return 0


def cmd_examples(a) -> int:
    for d in _data_dirs(a.data):
        cdir = os.path.join(d, "computations") if os.path.isdir(os.path.join(d, "computations")) else d
        if not os.path.isdir(cdir):
            continue
        for fn in sorted(os.listdir(cdir)):
            if not fn.endswith(".json"):
                continue
            with open(os.path.join(cdir, fn)) as f:
                j = json.load(f)
            if "dims" not in j:
                continue
            print(f"{j['name']}: dims {'x'.join(str(n) for n in j['sizes'])}, combine [{', '.join(j['combine'])}], "
                  f"{j['inputs'][0]['type']}")
        fdir = os.path.join(d, "fixtures")
        if os.path.isdir(fdir):
            for fn in sorted(os.listdir(fdir)):
                with open(os.path.join(fdir, fn)) as f:
                    fx = json.load(f)
                print(f"fixture {fx['name']}: {fx['spec']} on {fx['model']}")
        break
    return 0


def build_parser():
    ap = argparse.ArgumentParser(prog="mdh", description="Multi-dimensional homomorphism pipeline (B200 backend)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def source(p, config=True):
        p.add_argument("--spec", help="bundled computation name or spec JSON file")
        p.add_argument("--asm", default="B200", help="ASM preset name, inline JSON, or file (default B200)")
        if config:
            p.add_argument("--config", help="tuning configuration JSON file")
        p.add_argument("--data", help="reference data dir (computations/, fixtures/)")
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--device", type=int, default=0)

    v = sub.add_parser("verify", help="run configurations against the device reference executor")
    source(v)
    v.add_argument("--fixture", help="bundled fixture name or file (overrides spec/asm/config)")
    v.add_argument("--random", type=int, default=0, help="number of random configurations to sample (seeds seed + k)")
    t = sub.add_parser("tune", help="search the configuration space on the device")
    source(t, config=False)
    t.add_argument("--budget", type=int, default=20)
    t.add_argument("--objective", default="simcost", choices=["simcost", "compiled", "device"],
                   help="simcost (the reference's default, mdh_main.cpp:306): the input-free cost model; "
                        "compiled / device: CUDA-event time of the instantiated kernel on the B200")
    t.add_argument("--seed-simcost", action="store_true",
                   help="random phase samples the cheapest quarter of the candidates by SimCost")
    t.add_argument("--start", help="fixture (name or file) whose configuration is evaluated first")
    t.add_argument("--out")
    t.add_argument("--history")
    t.add_argument("--tf32", action="store_true")
    lw = sub.add_parser("lower", help="print the lowered expression (LowLevelExpr::pretty)")
    source(lw)
    lw.add_argument("--fixture", help="bundled fixture name or file (overrides spec/asm/config)")
    lw.add_argument("--out")
    e = sub.add_parser("emit", help="print the CUDA kernel compiled for the md_hom")
    source(e)
    e.add_argument("--out")
    e.add_argument("--f64", action="store_true", help="f64 storage (the bit-exact mode)")
    e.add_argument("--gate-compile", action="store_true",
                   help="run the compiled kernel on the driver's inputs against the device reference executor")
    d = sub.add_parser("describe", help="print the plan (family, template, Table-1 config)")
    source(d)
    d.add_argument("--tf32", action="store_true")
    r = sub.add_parser("run", help="execute on a ref-file's inputs, print outputs as JSON")
    source(r)
    r.add_argument("--inputs", required=True)
    r.add_argument("--out")
    x = sub.add_parser("examples", help="list bundled computations and fixtures")
    x.add_argument("--data")
    return ap


def main(argv=None) -> int:
    ap = build_parser()
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 3
    cmds = {"verify": cmd_verify, "tune": cmd_tune, "lower": cmd_lower, "emit": cmd_emit, "describe": cmd_describe,
            "run": cmd_run, "examples": cmd_examples}
    try:
        return cmds[a.cmd](a)
    except CliError as e:
        print(str(e), file=sys.stderr)
        return exit_code_for(e.code)
    except mdh.MdhError as e:
        print(str(e), file=sys.stderr)
        return exit_code_for(e.code)


if __name__ == "__main__":
    sys.exit(main())
