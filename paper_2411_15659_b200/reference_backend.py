"""The ``b200`` backends inside the reference package.

The reference selects backends by closed string dispatch in three places
(``estimator.BACKENDS``/``Conv2D._conv_one``, ``estimator.py:24, 99-110``;
``runner.BACKEND_ORDER``/``_backend_plan``, ``runner.py:33, 65-86``; the CLI
``--backend`` choices and ``_run_conv``, ``cli.py:41, 92-102``) and has no
plugin registry.  ``install(smmconv)`` applies to an UNMODIFIED, imported
reference package exactly the additions INTEGRATION.md describes for a
maintainer, so the reference's own harness (its runner with the checksum
guard and scratch meter, its CSV writer, its CLI and its estimator) drives
the B200 path beside its CPU backends:

* ``b200`` -- the fp32 FFMA product kernel; ``b200_exact`` -- the bitwise
  mode (equal to ``smm_conv_single`` bit for bit);
* both take the reference's numpy arrays through the host C-ABI entry
  ``smmc_conv2d_fwd_f32_host`` (H2D + kernel + D2H, synchronous, a fresh
  output array as ``smm.py:236``), validated by the reference's own
  ``check_input`` / ``check_weights_smm`` (``validation.py:25-50``);
* scratch: 0 elements of reference-metered scratch (the zero-packed slice
  lives in shared memory), which the runner verifies against its meter.

Only the dispatch is patched; every number, check and file format is the
reference's.  ``uninstall`` restores the originals.
"""

import ctypes

import numpy as np

from . import _native

__all__ = ["BACKENDS", "install", "uninstall", "smm_conv_b200"]

BACKENDS = ("b200", "b200_exact")
_MODE = {"b200": 0, "b200_exact": 1}
_SAVED = {}


def smm_conv_b200(smmconv, inp, weights_smm, geom, backend="b200"):
    """One sample (c_i, h, w) -> (c_o, h', w') through the C ABI, with the
    reference's validation and exception types (the INTEGRATION.md stub)."""
    smmconv.validation.check_input(inp, geom)
    smmconv.validation.check_weights_smm(weights_smm, geom)
    out = np.empty(geom.output_shape, dtype=np.float32)
    g = _native.Geom(1, geom.in_channels, geom.in_h, geom.in_w, geom.out_channels,
                     geom.k_h, geom.k_w, geom.stride_h, geom.stride_w, geom.pad_h, geom.pad_w)
    st = _native.lib().smmc_conv2d_fwd_f32_host(
        ctypes.c_void_p(inp.ctypes.data), ctypes.c_void_p(weights_smm.ctypes.data),
        ctypes.c_void_p(out.ctypes.data), ctypes.byref(g), _MODE[backend], _device())
    if st:
        errs = smmconv.errors
        exc = {_native.SMMC_EGEOM: errs.GeometryError,
               _native.SMMC_ESHAPE: errs.ShapeMismatchError}.get(st, errs.SmmConvError)
        raise exc(_native.last_error())
    return out


def _device():
    from .smm import _device as dev
    return dev()


def install(smmconv):
    """Add the b200 backends to an imported reference ``smmconv`` package."""
    if "runner" in _SAVED:
        return smmconv
    import importlib
    for sub in ("runner", "estimator", "cli", "validation", "errors", "smm", "workspace", "csvio",
                "layers"):
        importlib.import_module(f"{smmconv.__name__}.{sub}")
    runner, estimator, cli = smmconv.runner, smmconv.estimator, smmconv.cli
    _SAVED.update(runner=(runner.BACKEND_ORDER, runner._backend_plan),
                  estimator=(estimator.BACKENDS, estimator.Conv2D.fit,
                             estimator.Conv2D._conv_one),
                  cli=(cli.BACKEND_ORDER, cli._run_conv))
    orig_plan = runner._backend_plan

    # runner.py:65-86 -- "b200": (True, runner, 0 scratch elements)
    def _backend_plan(backend, geom, weights, weights_smm, threads, use_blas):
        if backend in BACKENDS:
            w_smm = weights_smm if weights_smm is not None else \
                smmconv.smm.repack_weights(weights, geom)
            return True, (lambda inp: smm_conv_b200(smmconv, inp, w_smm, geom, backend)), 0
        return orig_plan(backend, geom, weights, weights_smm, threads, use_blas)

    runner._backend_plan = _backend_plan
    runner.BACKEND_ORDER = tuple(runner.BACKEND_ORDER) + BACKENDS

    # estimator.py:24, 71-110 -- repack at fit, dispatch per sample
    orig_fit, orig_one = estimator.Conv2D.fit, estimator.Conv2D._conv_one
    estimator.BACKENDS = tuple(estimator.BACKENDS) + BACKENDS

    def fit(self, X, y=None):
        out = orig_fit(self, X, y)
        if self.backend in BACKENDS:
            self.weights_smm_ = smmconv.smm.repack_weights(self.weights_, self.geometry_)
        return out

    def _conv_one(self, image):
        if self.backend in BACKENDS:
            return smm_conv_b200(smmconv, image, self.weights_smm_, self.geometry_, self.backend)
        return orig_one(self, image)

    estimator.Conv2D.fit = fit
    estimator.Conv2D._conv_one = _conv_one

    # cli.py:41, 92-102 -- `smmconv conv --backend b200`
    orig_run_conv = cli._run_conv
    cli.BACKEND_ORDER = runner.BACKEND_ORDER

    def _run_conv(args):
        if args.backend not in BACKENDS:
            return orig_run_conv(args)
        geom = smmconv.ConvGeometry(
            in_channels=args.ci, out_channels=args.co, in_h=args.h, in_w=args.w,
            k_h=args.kh, k_w=args.kw, stride_h=args.sh, stride_w=args.sw,
            pad_h=args.ph, pad_w=args.pw)
        inp = smmconv.random_tensor(geom.input_shape, args.seed)
        weights = smmconv.random_tensor(geom.weights_shape, args.seed + 1)
        w_smm = smmconv.smm.repack_weights(weights, geom)
        with smmconv.workspace.metered() as meter:
            out = smm_conv_b200(smmconv, inp, w_smm, geom, args.backend)
        print(f"checksum={float(out.sum(dtype='float64'))!r}")
        print(f"scratch_bytes={meter.total_alloc_bytes(4)}")
        return 0

    cli._run_conv = _run_conv
    return smmconv


def uninstall(smmconv):
    if "runner" not in _SAVED:
        return
    smmconv.runner.BACKEND_ORDER, smmconv.runner._backend_plan = _SAVED.pop("runner")
    (smmconv.estimator.BACKENDS, smmconv.estimator.Conv2D.fit,
     smmconv.estimator.Conv2D._conv_one) = _SAVED.pop("estimator")
    smmconv.cli.BACKEND_ORDER, smmconv.cli._run_conv = _SAVED.pop("cli")
