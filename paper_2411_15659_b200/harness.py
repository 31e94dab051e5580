"""Benchmark harness on the GPU: the SURVEY §8(f) "next" rows.

GPU counterparts of the reference's harness pieces, same formats:

* layer configs — the reference's line format (``layers.py:1-11, 43-97``):
  ``layer name=<label> ci= co= h= w= kh= kw= [sh= sw= ph= pw=]``;
* the paper's four parameter sweeps (``layers.py:114-135``) and the three
  network presets (AlexNet, VGG-16 -- the BASELINE config 4 shapes -- and
  YOLOv3-tiny, ``layers.py:28, 100-106``) as data (``workloads.NETWORKS``);
  any other network is read from a .cfg file via ``load_layer_config``;
* ``run_bench`` (``runner.py:97-172``): deterministic splitmix64 inputs, one
  warm-up run, median of >= 3 CUDA-event-timed repeats, float64 checksums that
  must agree across backends (1e-3 relative; 2e-2 for the bf16 variant) or
  ``ChecksumMismatchError``, speedup against the im2col comparator;
* CSV with the reference's exact header and field formatting
  (``csvio.py:14-68``), byte-identical round trip;
* scratch accounting: ``scratch_bytes`` is the global-memory scratch a
  backend allocates per call — 0 for the fused SMM kernel (its zero-packed
  slice lives in shared memory), the split-K/stream-K workspace when used,
  the lowered matrix for im2col (the paper's memory claim, Eq. 1).

Backends: ``b200_smm`` (FFMA product), ``b200_exact`` (bitwise mode),
``b200_bf16_tc`` (tcgen05 bf16 variant, own tolerance), ``b200_bf16x3_tc``
(fp32-accurate split-bf16 tensor-core path, fp32 checksum bar), ``b200_im2col``
(explicit lowered matrix by a kernel of this library + a cuBLAS SGEMM with
TF32 off — a plain library GEMM, the paper's comparator).

    python -m paper_2411_15659_b200.harness --network vgg16 --csv out.csv
"""

import argparse
import statistics
import sys
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Optional

import numpy as np

from . import _native
from .errors import ChecksumMismatchError, ConfigError, GeometryError
from .geometry import ConvGeometry
from .tensors import random_tensor

__all__ = [
    "LayerSpec", "parse_layer_config", "load_layer_config", "sweep", "builtin_network",
    "BenchRecord", "run_bench", "emit_csv", "parse_csv", "CSV_HEADER", "BACKENDS",
    "SWEEP_KINDS", "NETWORK_NAMES",
]

BACKENDS = ("b200_im2col", "b200_smm", "b200_exact", "b200_bf16_tc", "b200_bf16x3_tc")
SWEEP_KINDS = ("in_channels", "spatial", "kernel", "out_channels")
CSV_HEADER = ("layer,backend,threads,repeats,median_time_s,scratch_bytes,"
              "speedup_vs_im2col,checksum")
_CHECKSUM_RTOL = 1e-3
_CHECKSUM_RTOL_BF16 = 2e-2

_FIELDS = {"ci": 1, "co": 1, "h": 1, "w": 1, "kh": 1, "kw": 1,
           "sh": 1, "sw": 1, "ph": 0, "pw": 0}  # minimum values
_REQUIRED = ("ci", "co", "h", "w", "kh", "kw")
_DEFAULTS = {"sh": 1, "sw": 1, "ph": 0, "pw": 0}


@dataclass(frozen=True)
class LayerSpec:
    name: str
    geometry: ConvGeometry


def _layer_from_line(line, lineno):
    tokens = line.split()
    if tokens[0] != "layer":
        raise ConfigError(f"line {lineno}: expected 'layer', got {tokens[0]!r}")
    raw = {}
    for tok in tokens[1:]:
        key, eq, val = tok.partition("=")
        if not eq or not val:
            raise ConfigError(f"line {lineno}: malformed field {tok!r}")
        if key in raw:
            raise ConfigError(f"line {lineno}: duplicate field {key!r}")
        raw[key] = val
    name = raw.pop("name", None)
    if not name:
        raise ConfigError(f"line {lineno}: missing field 'name'")
    vals = dict(_DEFAULTS)
    seen = set()
    for key, val in raw.items():
        if key not in _FIELDS:
            raise ConfigError(f"line {lineno}: unknown field {key!r}")
        try:
            vals[key] = int(val)
        except ValueError:
            raise ConfigError(f"line {lineno}: field {key!r} must be an integer, "
                              f"got {val!r}") from None
        seen.add(key)
    missing = [k for k in _REQUIRED if k not in seen]
    if missing:
        raise ConfigError(f"line {lineno}: missing field {missing[0]!r}")
    for key, v in vals.items():
        if v < _FIELDS[key]:
            raise ConfigError(f"line {lineno}: {key} must be >= {_FIELDS[key]}")
    try:
        geom = ConvGeometry(vals["ci"], vals["co"], vals["h"], vals["w"], vals["kh"],
                            vals["kw"], vals["sh"], vals["sw"], vals["ph"], vals["pw"])
    except GeometryError as exc:
        raise ConfigError(f"line {lineno}: {exc}") from exc
    return LayerSpec(name, geom)


def parse_layer_config(text):
    """Config text -> [LayerSpec]; '#' comments and blank lines skipped."""
    specs = []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if line:
            specs.append(_layer_from_line(line, lineno))
    return specs


def load_layer_config(path):
    return parse_layer_config(Path(path).read_text())


NETWORK_NAMES = ("alexnet", "vgg16", "yolov3")


def builtin_network(name):
    """Convolutional layers of a named architecture (the reference's presets,
    ``layers.py:100-106``; tables in ``workloads.NETWORKS``)."""
    if name not in NETWORK_NAMES:
        raise ConfigError(f"unknown network {name!r}; available: {', '.join(NETWORK_NAMES)}")
    from .workloads import network_geometries
    return [LayerSpec(nm, g) for nm, g in network_geometries(name)]


def _sq(ci, co, size, k):
    return ConvGeometry(ci, co, size, size, k, k)


def sweep(kind):
    """The paper's parameter sweeps (stride 1, no padding)."""
    if kind == "in_channels":
        return [LayerSpec(f"ci{ci}_hw{s}", _sq(ci, 32, s, 3))
                for ci in (1, 16, 32, 64, 128, 256) for s in (32, 64)]
    if kind == "spatial":
        return [LayerSpec(f"hw{s}_ci{ci}", _sq(ci, 32, s, 3))
                for ci in (1, 32, 64) for s in (32, 64, 128, 256, 512)]
    if kind == "kernel":
        return [LayerSpec(f"k{k}_hw{s}", _sq(32, 32, s, k))
                for k in (3, 5, 7, 9, 11, 13, 15) for s in (64, 256)]
    if kind == "out_channels":
        return [LayerSpec(f"co{co}", _sq(16, co, 256, 3)) for co in (1, 8, 16, 32, 64, 128)]
    raise ConfigError(f"unknown sweep {kind!r}; available: {', '.join(SWEEP_KINDS)}")


@dataclass(frozen=True)
class BenchRecord:
    layer: str
    backend: str
    threads: int
    repeats: int
    median_time_s: Optional[float]
    scratch_bytes: int
    speedup_vs_im2col: Optional[float]
    checksum: Optional[float]

    @property
    def unsupported(self):
        return self.median_time_s is None


# ------------------------------------------------------------------ backends
def _backend(name, geom, batch, x, w_oihw):
    """(supported, run() -> output tensor, scratch_bytes) on the current device."""
    import torch
    from . import device
    if name in ("b200_smm", "b200_exact"):
        mode = "ffma" if name == "b200_smm" else "exact"
        mod = device.SmmConv2d(geom, w_oihw, mode=mode, max_batch=batch)
        out = torch.empty((batch,) + geom.output_shape, device=x.device)
        scratch = _native.workspace_bytes(geom, batch, mode)
        return True, (lambda: mod(x, out=out)), scratch
    if name == "b200_bf16_tc":
        if not device.tc_supported(geom, batch):
            return False, None, 0
        mod = device.TcSmmConv2d(geom, w_oihw)
        xb = torch.empty(device.packed_input_shape(geom, batch), dtype=torch.bfloat16,
                         device=x.device)
        out = torch.empty((batch,) + geom.output_shape, device=x.device)
        scratch = xb.numel() * 2  # zero-padded channels-last bf16 copy of the input

        def run():
            mod(mod.pack_input(x, out=xb), out=out)
            return out
        return True, run, scratch
    if name == "b200_bf16x3_tc":  # fp32-accurate split-bf16 tensor-core path
        if not device.tc_supported(geom, batch):
            return False, None, 0
        mod = device.Tc3SmmConv2d(geom, w_oihw)
        out = torch.empty((batch,) + geom.output_shape, device=x.device)
        # the [hi|lo|hi] bf16 channels-last input copy + split-K partial planes
        scratch = (2 * 3 * batch * geom.padded_h * geom.padded_w * geom.in_channels +
                   device.tc_workspace_bytes(geom, batch, split3=True))
        return True, (lambda: mod(x, out=out)), scratch
    if name == "b200_im2col":
        import ctypes
        g = _native.Geom.of(geom, batch)
        nbytes = int(_native.lib().smmc_im2col_bytes(ctypes.byref(g)))
        kdim = geom.in_channels * geom.k_h * geom.k_w
        ohw = geom.out_h * geom.out_w
        low = torch.empty((batch, kdim, ohw), device=x.device)
        wmat = torch.as_tensor(w_oihw).reshape(geom.out_channels, kdim).to(x.device)
        out = torch.empty((batch, geom.out_channels, ohw), device=x.device)

        def run():
            stream = torch.cuda.current_stream(x.device).cuda_stream
            _native.check(_native.lib().smmc_im2col_pack_f32(
                ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(low.data_ptr()), ctypes.byref(g),
                ctypes.c_void_p(stream) if stream else None), "smmc_im2col_pack_f32")
            torch.matmul(wmat, low, out=out)  # cuBLAS SGEMM, TF32 disabled by run_bench
            return out.view((batch,) + geom.output_shape)
        return True, run, nbytes
    raise ValueError(f"unknown backend {name!r}; available: {', '.join(BACKENDS)}")


def _time(run, repeats):
    import torch
    run()
    torch.cuda.synchronize()
    times = []
    for _ in range(repeats):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = run()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) / 1e3)
    return statistics.median(times), out


def _rel(a, b):
    return abs(a - b) / max(abs(a), abs(b), 1e-12)


def run_bench(specs, backends, repeats=5, batch=1, seed=0):
    """One BenchRecord per (spec, backend), nested in that order."""
    import torch
    if repeats < 3:
        raise ValueError("repeats must be >= 3")
    for b in backends:
        if b not in BACKENDS:
            raise ValueError(f"unknown backend {b!r}; available: {', '.join(BACKENDS)}")
    if not torch.cuda.is_available():
        from .errors import DeviceError
        raise DeviceError("run_bench needs a CUDA device (no CPU fallback)")
    tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    records = []
    try:
        for spec in specs:
            g = spec.geometry
            # same deterministic fill as the reference harness (runner.py:118-121)
            x = torch.from_numpy(random_tensor((batch,) + g.input_shape, seed)).cuda()
            w = random_tensor(g.weights_shape, seed + 1)
            recs, sums = [], {}
            for name in backends:
                ok, run, scratch = _backend(name, g, batch, x, w)
                if not ok:
                    recs.append(BenchRecord(spec.name, name, sms, repeats, None, 0, None, None))
                    continue
                t, out = _time(run, repeats)
                sums[name] = float(out.double().sum().item())
                recs.append(BenchRecord(spec.name, name, sms, repeats, t, int(scratch), None,
                                        sums[name]))
            names = list(sums)
            for other in names[1:]:
                tol = (_CHECKSUM_RTOL_BF16 if "b200_bf16_tc" in (names[0], other)
                       else _CHECKSUM_RTOL)  # the split-bf16 path meets the fp32 bar
                if _rel(sums[names[0]], sums[other]) > tol:
                    raise ChecksumMismatchError(
                        f"checksum divergence on layer {spec.name!r}: {names[0]}="
                        f"{sums[names[0]]!r} vs {other}={sums[other]!r}")
            base = next((r.median_time_s for r in recs
                         if r.backend == "b200_im2col" and not r.unsupported), None)
            for r in recs:
                if base is not None and not r.unsupported:
                    r = replace(r, speedup_vs_im2col=base / r.median_time_s)
                records.append(r)
    finally:
        torch.backends.cuda.matmul.allow_tf32 = tf32
    return records


# ------------------------------------------------------------------ CSV
def _row(r):
    med = "" if r.median_time_s is None else f"{r.median_time_s:.6f}"
    spd = "" if r.speedup_vs_im2col is None else f"{r.speedup_vs_im2col:.4f}"
    chk = "" if r.checksum is None else repr(r.checksum)
    return f"{r.layer},{r.backend},{r.threads},{r.repeats},{med},{r.scratch_bytes},{spd},{chk}"


def emit_csv(records, destination=None):
    if not records:
        raise ValueError("no records to emit")
    text = "\n".join([CSV_HEADER] + [_row(r) for r in records]) + "\n"
    if destination is not None:
        if hasattr(destination, "write"):
            destination.write(text)
        else:
            Path(destination).write_text(text, encoding="ascii")
    return text


def _opt(tok, conv):
    return None if tok == "" else conv(tok)


def parse_csv(text):
    lines = text.splitlines()
    if not lines or lines[0] != CSV_HEADER:
        raise ConfigError("missing or unexpected CSV header")
    out = []
    for lineno, line in enumerate(lines[1:], start=2):
        f = line.split(",")
        if len(f) != 8:
            raise ConfigError(f"line {lineno}: expected 8 fields, got {len(f)}")
        try:
            out.append(BenchRecord(f[0], f[1], int(f[2]), int(f[3]), _opt(f[4], float),
                                   int(f[5]), _opt(f[6], float), _opt(f[7], float)))
        except ValueError as exc:
            raise ConfigError(f"line {lineno}: {exc}") from None
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(prog="paper_2411_15659_b200.harness")
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--network", choices=NETWORK_NAMES)
    src.add_argument("--config", help="layer config file (reference .cfg format)")
    src.add_argument("--sweep", choices=SWEEP_KINDS)
    ap.add_argument("--backends", default=",".join(BACKENDS))
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--csv", default="")
    ap.add_argument("--autotune", action="store_true",
                    help="per-shape autotuning of the b200_smm plans at fit (same as SMMC_AUTOTUNE=1)")
    a = ap.parse_args(argv)
    if a.autotune:
        import os
        os.environ["SMMC_AUTOTUNE"] = "1"
    specs = (builtin_network(a.network) if a.network else
             load_layer_config(a.config) if a.config else sweep(a.sweep))
    recs = run_bench(specs, a.backends.split(","), a.repeats, a.batch, a.seed)
    text = emit_csv(recs, a.csv or None)
    sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
