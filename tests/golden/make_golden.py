"""Generate tests/golden/smm_golden.npz from the REFERENCE implementation.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Every output array here is produced by the reference's own code —
``smmconv.smm_conv_single`` / ``smm_conv_parallel`` (smm.py:226-306),
``smmconv.conv_ref`` (reference.py:41-51), ``smmconv.extract_slice``
(smm.py:190-203) and ``smmconv.random_tensor`` (tensors.py:60-62) — so the
fixtures pin both our CPU oracle (tests/test_oracle.py) and the GPU kernels
(tests/test_gpu_parity.py) to the reference bit for bit.

Cases:
  * the reference's known-answer tests, restated as inputs/outputs
    (test_smm.py:171-184, test_reference.py:9-24, 68-72);
  * 12 small random geometries drawn like the reference's sample_geometry
    (conftest.py:52-70), splitmix64 data;
  * 20 geometries drawn like acceptance criterion 1 (test_acceptance.py:52-99);
  * BASELINE.json layer *types* at reduced channel counts with the BASELINE
    value distributions (x ~ U[-1,1), He-normal weights): 3x3 s1 p1 at the
    56/28/14/7 planes, 7x7 s2 p3, 11x11 s4 at 227x227, 5x5 p2 at 27, 1x1, plus
    ragged/rectangular/odd-channel edge cases;
  * zero-packed slices for a strided, padded geometry (test_smm.py:83-92);
  * the splitmix64 stream head (test_tensors.py:6-26).
"""

import json
import sys
from pathlib import Path

import numpy as np

import smmconv
from smmconv import (ConvGeometry, conv_ref, extract_slice, random_tensor,
                     repack_weights, smm_conv_parallel, smm_conv_single)

OUT = Path(__file__).resolve().parent / "smm_golden.npz"


def geom_tuple(g):
    return [g.in_channels, g.out_channels, g.in_h, g.in_w, g.k_h, g.k_w,
            g.stride_h, g.stride_w, g.pad_h, g.pad_w]


def he_normal(rng, g):
    std = np.float32(np.sqrt(2.0 / (g.in_channels * g.k_h * g.k_w)))
    w = rng.standard_normal(g.weights_shape, dtype=np.float32)
    return w * std


def main():
    arrays = {}
    manifest = []

    def add(name, g, x, w, kind):
        # x: (n, c_i, h, w) batch; the reference is single-sample, so loop.
        w_smm = repack_weights(w, g)
        ys, yr = [], []
        for xi in x:
            xi = np.ascontiguousarray(xi)
            a = smm_conv_single(xi, w_smm, g)
            b = smm_conv_parallel(xi, w_smm, g, 3)
            assert np.array_equal(a, b)
            ys.append(a)
            yr.append(conv_ref(xi, w, g))
        arrays[f"{name}__x"] = x
        arrays[f"{name}__w"] = w
        arrays[f"{name}__y_smm"] = np.stack(ys)
        arrays[f"{name}__y_ref"] = np.stack(yr)
        manifest.append({"name": name, "geom": geom_tuple(g), "n": int(x.shape[0]),
                         "kind": kind})

    # ---- known-answer tests (reference test_smm.py / test_reference.py)
    g = ConvGeometry(1, 1, 4, 4, 3, 3)
    add("kat_all_ones", g, np.ones((1,) + g.input_shape, np.float32),
        np.ones(g.weights_shape, np.float32), "kat")
    g = ConvGeometry(1, 1, 5, 6, 1, 1)
    add("kat_1x1_scaled_copy", g, random_tensor((1,) + g.input_shape, 5),
        np.full(g.weights_shape, 0.625, np.float32), "kat")
    g = ConvGeometry(1, 1, 6, 5, 3, 3)
    w = np.zeros(g.weights_shape, np.float32)
    w[0, 0, 0, 0] = 1.0
    add("kat_delta_crop", g, random_tensor((1,) + g.input_shape, 3), w, "kat")
    g = ConvGeometry(2, 3, 6, 6, 3, 3, pad_h=1, pad_w=1)
    add("kat_zero_weights", g, random_tensor((1,) + g.input_shape, 4),
        np.zeros(g.weights_shape, np.float32), "kat")

    # ---- small random geometries (conftest.sample_geometry grid)
    rng = np.random.default_rng(1234)
    i = 0
    while i < 12:
        kw = dict(in_channels=int(rng.integers(1, 5)), out_channels=int(rng.integers(1, 5)),
                  in_h=int(rng.integers(4, 13)), in_w=int(rng.integers(4, 13)),
                  k_h=int(rng.choice((1, 3, 5))), k_w=int(rng.choice((1, 3, 5))),
                  stride_h=int(rng.choice((1, 2))), stride_w=int(rng.choice((1, 2))),
                  pad_h=int(rng.choice((0, 1))), pad_w=int(rng.choice((0, 1))))
        if kw["k_h"] > kw["in_h"] + 2 * kw["pad_h"] or kw["k_w"] > kw["in_w"] + 2 * kw["pad_w"]:
            continue
        g = ConvGeometry(**kw)
        add(f"rand_small_{i:02d}", g, random_tensor((2,) + g.input_shape, 5 * i),
            random_tensor(g.weights_shape, 5 * i + 1), "random")
        i += 1

    # ---- acceptance-criterion-1 style geometries
    rng = np.random.default_rng(20240601)
    i = 0
    while i < 20:
        kw = dict(in_channels=int(rng.integers(1, 9)), out_channels=int(rng.integers(1, 9)),
                  in_h=int(rng.integers(4, 33)), in_w=int(rng.integers(4, 33)),
                  k_h=int(rng.choice((1, 3, 5, 7))), k_w=int(rng.choice((1, 3, 5, 7))),
                  stride_h=int(rng.choice((1, 2))), stride_w=int(rng.choice((1, 2))),
                  pad_h=int(rng.choice((0, 1, 2))), pad_w=int(rng.choice((0, 1, 2))))
        if kw["k_h"] > kw["in_h"] + 2 * kw["pad_h"] or kw["k_w"] > kw["in_w"] + 2 * kw["pad_w"]:
            continue
        g = ConvGeometry(**kw)
        add(f"accept_{i:02d}", g, random_tensor((1,) + g.input_shape, 2 * i + 2),
            random_tensor(g.weights_shape, 2 * i + 3), "acceptance")
        i += 1

    # ---- BASELINE.json layer types, reduced channels, BASELINE distributions
    layer_cases = [
        ("cfg1_3x3_c8_56", (8, 8, 56, 56, 3, 3, 1, 1, 1, 1), 1),
        ("cfg2_3x3_c16_28", (16, 16, 28, 28, 3, 3, 1, 1, 1, 1), 2),
        ("cfg2_3x3_c24_14", (24, 24, 14, 14, 3, 3, 1, 1, 1, 1), 2),
        ("cfg2_3x3_c40_7", (40, 40, 7, 7, 3, 3, 1, 1, 1, 1), 3),
        ("cfg3_7x7s2p3_3to8_40", (3, 8, 40, 40, 7, 7, 2, 2, 3, 3), 2),
        ("cfg3_11x11s4_3to8_227", (3, 8, 227, 227, 11, 11, 4, 4, 0, 0), 1),
        ("cfg3_5x5p2_12to16_27", (12, 16, 27, 27, 5, 5, 1, 1, 2, 2), 1),
        ("cfg3_1x1_32to8_28", (32, 8, 28, 28, 1, 1, 1, 1, 0, 0), 2),
        ("cfg4_3x3_3to16_48", (3, 16, 48, 48, 3, 3, 1, 1, 1, 1), 1),
        ("cfg5_1x1_8to40_14", (8, 40, 14, 14, 1, 1, 1, 1, 0, 0), 2),
        ("edge_rect_3x5_s2x1_p1x2", (5, 7, 13, 17, 3, 5, 2, 1, 1, 2), 2),
        ("edge_odd_co5_s3", (3, 5, 19, 23, 3, 3, 3, 3, 1, 0), 2),
        ("edge_ci1_co1_1x1", (1, 1, 9, 11, 1, 1, 1, 1, 0, 0), 3),
        ("edge_kernel_eq_padded", (4, 6, 5, 5, 7, 7, 1, 1, 1, 1), 2),
        ("edge_co130_tile_tail", (9, 130, 6, 6, 3, 3, 1, 1, 1, 1), 2),
    ]
    for idx, (name, gt, n) in enumerate(layer_cases):
        g = ConvGeometry(*gt)
        rng = np.random.default_rng(7000 + idx)
        x = rng.random((n,) + g.input_shape, dtype=np.float32) * np.float32(2) - np.float32(1)
        add(name, g, x, he_normal(rng, g), "baseline_type")

    # ---- zero-packed slices (test_smm.py:83-92 geometry)
    g = ConvGeometry(2, 1, 6, 5, 3, 3, stride_w=2, pad_h=2, pad_w=1)
    x = random_tensor(g.input_shape, 3)
    arrays["slices__x"] = x
    for c in range(g.in_channels):
        for j in range(g.k_w):
            buf = np.empty((g.padded_h, g.out_w), np.float32)
            extract_slice(x, g, c, j, buf)
            arrays[f"slices__c{c}_j{j}"] = buf.copy()
    manifest.append({"name": "slices", "geom": geom_tuple(g), "n": 1, "kind": "slices"})

    # ---- splitmix64 head
    arrays["splitmix__seed42_head4"] = random_tensor(4, 42)
    arrays["splitmix__seed7_3x4x5"] = random_tensor((3, 4, 5), 7)

    arrays["manifest"] = np.array(json.dumps({
        "generator": "tests/golden/make_golden.py",
        "reference": f"smmconv {smmconv.__version__} (/root/reference/pkg)",
        "cases": manifest}))
    np.savez_compressed(OUT, **arrays)
    total = sum(a.nbytes for a in arrays.values())
    print(f"wrote {OUT} ({len(manifest)} cases, {total / 1e6:.2f} MB raw, "
          f"{OUT.stat().st_size / 1e6:.2f} MB on disk)")


if __name__ == "__main__":
    sys.exit(main())
