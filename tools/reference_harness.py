"""Drive the B200 path from the reference's OWN harness:
install the ``b200`` backends into the unmodified reference package from
baseline/_ref (paper_2411_15659_b200.reference_backend, the INTEGRATION.md
stub) and run the reference's CLI ``smmconv bench`` -- its runner (median of
timed repeats, float64 checksums that must agree across backends within
1e-3, scratch verified against its meter), its CSV writer -- on the network
presets and the paper's sweeps, CPU backends beside ``b200``.

    python tools/reference_harness.py --outdir profiles/r02/reference_harness
"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/smmc_numba_cache")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--outdir", default="gpurun_out/reference_harness")
    ap.add_argument("--runs", default="vgg16:im2col,smm,b200,b200_exact;"
                                      "alexnet:ref,im2col,mec,smm,b200,b200_exact;"
                                      "yolov3:im2col,mec,smm,b200;"
                                      "sweep=in_channels:im2col,smm,b200;sweep=kernel:im2col,smm,b200")
    ap.add_argument("--repeats", default="3")
    a = ap.parse_args()
    import smmconv
    import smmconv.cli

    from paper_2411_15659_b200 import reference_backend
    reference_backend.install(smmconv)
    out = Path(a.outdir)
    out.mkdir(parents=True, exist_ok=True)
    for run in a.runs.split(";"):
        src, backends = run.split(":")
        if src.startswith("sweep="):
            args, tag = ["--sweep", src[6:]], "sweep_" + src[6:]
        else:
            args, tag = ["--network", src], src
        dest = out / f"{tag}.csv"
        rc = smmconv.cli.main(["bench", *args, "--backends", backends, "--repeats", a.repeats,
                               "--out", str(dest)])
        print(f"{tag}: rc={rc} -> {dest}", flush=True)
        if rc:
            return rc
    return 0


if __name__ == "__main__":
    sys.exit(main())
