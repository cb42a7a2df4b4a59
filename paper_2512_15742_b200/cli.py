"""GPU backend for the reference CLI's forward-path commands (SURVEY §8 row
f2; proj/tools/main.cpp): ``run`` (cmd_run, main.cpp:265-302), ``bench``
(cmd_bench, 304-345) and ``inspect`` (header + memory plan).  Same options,
defaults (batch 64, repeats 101, warmup 10), output files (outputs.csv in
%.17g, bench.csv from bench_csv, manifest.txt), stdout lines and exit codes
(0 ok; 1 usage/config; 2 model file / validation; 3 internal,
main.cpp:616-637).  The models are loaded straight into HBM
(skan_head_load_file) and evaluated on the GPU.

    python -m paper_2512_15742_b200 run --model m.skan --input x.csv [--out-dir D]
    python -m paper_2512_15742_b200 bench --model a.skan --model b.skan [--batch 64 --repeats 101 --warmup 10 --seed S]
    python -m paper_2512_15742_b200 inspect --model m.skan
"""
from __future__ import annotations

import argparse
import builtins
import os
import sys
from typing import List, Optional

import numpy as np

from . import errors
from .lutham import BenchConfig, bench_csv, bench_iso_latency, compressed_forward, load_model, make_workspace

TOOL_VERSION = "1.0.0"  # main.cpp:25 (the manifest's tool line)


class ConfigError(errors.HoloquantError):
    """holoquant::ConfigError (exit code 1)."""


def _worker_count() -> int:
    """analysis.cpp:17-24: HOLOQUANT_THREADS in [1, 256], else 1."""
    env = os.environ.get("HOLOQUANT_THREADS", "")
    v = int(env) if env.isdigit() or (env[:1] in "+-" and env[1:].isdigit()) else 0
    return v if 1 <= v <= 256 else 1


_WS = " \t\n\v\f\r"


def _stod_cell(cell: str) -> float:
    """std::stod plus main.cpp's check that only whitespace follows the number."""
    t = cell.lstrip(_WS).rstrip(_WS)
    if not t or "_" in t:
        raise builtins.ValueError(cell)
    try:
        return float(t)
    except builtins.ValueError:
        if t.lstrip("+-")[:2].lower() != "0x":
            raise
        return float.fromhex(t)  # stod reads 0x hex floats too


def _format_full(v: float) -> str:
    return "%.17g" % v


def _format3(v: float) -> str:
    return "%.3f" % v


def _write_manifest(d: str, command: str, fields: List[tuple]) -> None:
    m = f"tool = holoquant {TOOL_VERSION}\ncommand = {command}\n"
    for k, v in fields:
        m += f"{k} = {v}\n"
    m += f"threads = {_worker_count()}\n"
    with open(os.path.join(d, "manifest.txt"), "w") as f:
        f.write(m)


def _prepare_out_dir(d: str) -> str:
    os.makedirs(d, exist_ok=True)
    return d


def _parse_input_csv(path: str, width: int) -> np.ndarray:
    """parse_input_csv (main.cpp:222-262): comma-separated doubles per line,
    blank lines skipped, each row exactly `width` values."""
    try:
        f = open(path, "r", newline="")
    except OSError:
        raise errors.ValueError(f"cannot open '{path}'")
    rows = []
    with f:
        for line_no, line in enumerate(f.read().split("\n"), start=1):
            if line.endswith("\r"):
                line = line[:-1]
            if not line.strip():
                continue
            row = []
            for cell in line.split(","):
                try:
                    row.append(_stod_cell(cell))
                except builtins.ValueError:
                    raise errors.ValueError(f"row {line_no}: cannot parse '{cell}' as a number")
            if len(row) != width:
                raise errors.ValueError(f"row {line_no}: expected {width} values, got {len(row)}")
            rows.append(row)
    return np.asarray(rows, dtype=np.float64).reshape(len(rows), width)


def cmd_run(model_path: str, input_path: str, out_dir: str, mode: str = "exact") -> int:
    model = load_model(model_path)
    rows = _parse_input_csv(input_path, model.input_dim())
    batch = rows.shape[0]
    out = model.output_dim()
    outputs = np.zeros(batch * out, dtype=np.float64)
    if batch:
        ws = make_workspace(model, batch)
        compressed_forward(model, rows.reshape(-1), batch, outputs, ws, mode=mode)
    csv = "".join(",".join(_format_full(v) for v in outputs[r * out:(r + 1) * out]) + "\n" for r in range(batch))
    d = _prepare_out_dir(out_dir)
    with open(os.path.join(d, "outputs.csv"), "w") as f:
        f.write(csv)
    _write_manifest(d, "run", [("model", model_path), ("input", input_path), ("rows", str(batch)),
                               ("outputs", "outputs.csv")])
    print(f"wrote {batch} output rows to {os.path.join(d, 'outputs.csv')}")
    return 0


def cmd_bench(model_paths: List[str], batch: int, repeats: int, warmup: int, seed: Optional[int],
              out_dir: str, mode: str = "exact") -> int:
    if len(model_paths) < 2:
        raise ConfigError("bench needs at least two --model files")
    models = [load_model(p) for p in model_paths]
    bc = BenchConfig(batch=batch, repeats=repeats, warmup=warmup,
                     seed=seed if seed is not None else BenchConfig().seed)
    rows = bench_iso_latency(models, bc, mode=mode)
    lo = min(r.median_us for r in rows)
    hi = max(r.median_us for r in rows)
    for r in rows:
        print(f"G={r.grid_size}: median {_format3(r.median_us)} us, IQR [{_format3(r.p25_us)}, {_format3(r.p75_us)}]")
    print(f"max/min median ratio: {_format3(hi / lo)}")
    d = _prepare_out_dir(out_dir)
    with open(os.path.join(d, "bench.csv"), "w") as f:
        f.write(bench_csv(rows))
    _write_manifest(d, "bench", [("models", " ".join(model_paths)), ("batch", str(batch)), ("repeats", str(repeats)),
                                 ("warmup", str(warmup)), ("seed", str(bc.seed)), ("outputs", "bench.csv")])
    return 0


def cmd_inspect(model_path: str) -> int:
    model = load_model(model_path)
    plan = model.plan()
    print(f"layers: {len(model.layers)}  input {model.input_dim()}  output {model.output_dim()}")
    for i, h in enumerate(model.layers):
        print(f"layer {i}: {h.in_dim}->{h.out_dim} G={h.grid_size} K={h.k} domain [{_format_full(h.domain_lo)}, "
              f"{_format_full(h.domain_hi)}]")
    print(f"payload {plan.payload_total} B, working set {plan.working_set_total} B, device {plan.device_total} B")
    return 0


def main(argv: Optional[List[str]] = None) -> int:
    ap = argparse.ArgumentParser(prog="holoquant-b200", description="spline-network VQ toolkit, B200 backend")
    sub = ap.add_subparsers(dest="cmd")

    def common(p):
        p.add_argument("--seed", type=int, default=None, help="seed override")
        p.add_argument("--out-dir", default=".", help="output directory")
        p.add_argument("--mode", choices=["exact", "fast"], default="exact",
                       help="exact: the reference's f64 arithmetic, bitwise (default); fast: f32 edges")

    p_run = sub.add_parser("run", help="evaluate a model on CSV inputs")
    p_run.add_argument("--model", required=True)
    p_run.add_argument("--input", required=True)
    common(p_run)
    p_bench = sub.add_parser("bench", help="latency comparison across grid sizes")
    p_bench.add_argument("--model", action="append", required=True)
    p_bench.add_argument("--batch", type=int, default=64)
    p_bench.add_argument("--repeats", type=int, default=101)
    p_bench.add_argument("--warmup", type=int, default=10)
    common(p_bench)
    p_ins = sub.add_parser("inspect", help="dump model header and memory plan")
    p_ins.add_argument("--model", required=True)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # CLI::ParseError: --help is 0, anything else 1 (main.cpp:596-599)
        return 0 if e.code == 0 else 1
    if a.cmd is None:
        ap.print_usage(sys.stderr)
        return 1
    try:
        if a.cmd == "run":
            return cmd_run(a.model, a.input, a.out_dir, a.mode)
        if a.cmd == "bench":
            return cmd_bench(a.model, a.batch, a.repeats, a.warmup, a.seed, a.out_dir, a.mode)
        return cmd_inspect(a.model)
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return 1
    except errors.FormatError as e:
        print(f"model file error: {e}", file=sys.stderr)
        return 2
    except (errors.ShapeError, errors.ValueError) as e:
        print(f"validation error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # noqa: BLE001 - main.cpp:633 catches std::exception
        print(f"internal error: {e}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
