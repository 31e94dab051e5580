"""the reference's OWN harness drives the B200 path.

``reference_backend.install`` adds the ``b200`` / ``b200_exact`` backends to
the unmodified reference package installed under baseline/_ref (the
INTEGRATION.md stub); then the reference's runner (checksum guard across
backends, scratch verified against its meter, CSV), its estimator and its
CLI run them beside the CPU backends."""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "smmconv").exists(),
                                 reason="reference not installed under baseline/_ref")]


@pytest.fixture(scope="module")
def smmconv():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/smmc_numba_cache")
    sys.path.insert(0, str(REF))
    import smmconv as ref

    from paper_2411_15659_b200 import reference_backend
    reference_backend.install(ref)
    yield ref
    reference_backend.uninstall(ref)


def test_reference_runner_alexnet_all_backends(smmconv):
    """Criterion 6 of the reference (test_acceptance.py:191-205) with the
    b200 backends added: fixed row count incl. the unsupported pair, the
    runner's checksum guard passes, b200 scratch is 0 metered elements."""
    from smmconv.layers import builtin_network
    from smmconv.runner import run_bench
    backends = ["ref", "im2col", "mec", "smm", "b200", "b200_exact"]
    recs = run_bench(builtin_network("alexnet"), backends, repeats=3, threads=2, seed=1)
    assert len(recs) == 5 * len(backends)
    by = {}
    for r in recs:
        by.setdefault(r.layer, {})[r.backend] = r
    assert by["conv1"]["mec"].unsupported and not by["conv1"]["b200"].unsupported
    for layer, rs in by.items():
        assert rs["b200"].scratch_bytes == 0 and rs["b200_exact"].scratch_bytes == 0
        # exact mode reproduces the reference's smm checksum bit for bit
        assert rs["b200_exact"].checksum == rs["smm"].checksum, layer
        assert abs(rs["b200"].checksum - rs["smm"].checksum) <= 1e-5 * abs(rs["smm"].checksum)
        assert rs["b200"].speedup_vs_im2col is not None


def test_reference_csv_roundtrip_with_b200_rows(smmconv):
    from smmconv.csvio import emit_csv, parse_csv
    from smmconv.layers import sweep
    from smmconv.runner import run_bench
    recs = run_bench(sweep("out_channels")[:3], ["smm", "b200"], repeats=3, threads=2, seed=3)
    text = emit_csv(recs)
    assert emit_csv(parse_csv(text)) == text
    assert sum(",b200," in ln for ln in text.splitlines()) == 3


def test_reference_estimator_b200(smmconv):
    X = smmconv.random_tensor((3, 5, 12, 11), 4)
    kw = dict(out_channels=6, kernel_size=(3, 5), stride=(1, 2), padding=(1, 2), seed=8)
    y_smm = smmconv.Conv2D(backend="smm", **kw).fit(X).transform(X)
    y_ex = smmconv.Conv2D(backend="b200_exact", **kw).fit(X).transform(X)
    y_ff = smmconv.Conv2D(backend="b200", **kw).fit(X).transform(X)
    assert np.array_equal(y_ex, y_smm)
    assert smmconv.max_rel_diff(y_ff, y_smm) <= 1e-4


def test_reference_cli_conv_b200(smmconv, capsys):
    from smmconv.cli import main
    args = ["conv", "--ci", "16", "--co", "32", "--h", "64", "--w", "64", "--kh", "3", "--kw", "3"]
    assert main(args + ["--backend", "smm"]) == 0
    smm_out = capsys.readouterr().out
    assert main(args + ["--backend", "b200_exact"]) == 0
    b_out = capsys.readouterr().out
    # bitwise equal checksum; 0 B of metered scratch (the reference's smm: 1 slice buffer)
    assert smm_out.splitlines()[0] == b_out.splitlines()[0]
    assert b_out.splitlines()[1] == "scratch_bytes=0"
