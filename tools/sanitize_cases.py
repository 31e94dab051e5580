#!/usr/bin/env python
"""Small launches of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), one tool per box call:

    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_cases.py

Each case forces one work decomposition or kernel (SMMC_FORCE_PLAN and the
other A/B hooks are read per call) on a tiny geometry, runs it, checks it
against the CPU oracle (so a sanitizer-clean but wrong launch also fails) and
prints one line.  ``--only NAME`` runs the cases whose name contains NAME.
"""

import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--repeat", type=int, default=1,
                    help="race hunt: relaunch each FFMA case this many times into a NaN-poisoned "
                         "output (and, with --noise, beside a concurrent stream of unrelated "
                         "kernels that perturbs CTA scheduling); every result must be bitwise "
                         "equal to the first")
    ap.add_argument("--noise", action="store_true")
    args = ap.parse_args()

    import torch

    from oracle import smm_oracle as orc
    from paper_2411_15659_b200 import ConvGeometry, _native, device, repack_weights
    from paper_2411_15659_b200.parallel import cout_geometry, cout_shard
    from paper_2411_15659_b200.tensors import synthetic_layer

    torch.cuda.set_device(0)

    def G(ci, co, h, w, k, s=1, p=None):
        return ConvGeometry(ci, co, h, w, k, k, s, s, k // 2 if p is None else p,
                            k // 2 if p is None else p)

    def ffma(name, g, n, env, mode="ffma", tol=1e-4):
        return (name, "ffma", g, n, env, mode, tol)

    g3 = G(64, 96, 10, 10, 3)
    cases = [
        ffma("tiled_nosplit", g3, 2, {"SMMC_FORCE_PLAN": "0,1"}),
        ffma("tiled_64x128", g3, 2, {"SMMC_FORCE_PLAN": "3,1"}),
        ffma("splitk_last_arriver", g3, 2, {"SMMC_FORCE_PLAN": "1,3", "SMMC_CLUSTER_RED": "0"}),
        ffma("splitk_cluster_dsmem", g3, 1, {"SMMC_FORCE_PLAN": "1,2", "SMMC_CLUSTER_RED": "1"}),
        ffma("splitk_reduce_kernel", g3, 2, {"SMMC_FORCE_PLAN": "1,8", "SMMC_CLUSTER_RED": "0"}),
        ffma("streamk", g3, 2, {"SMMC_FORCE_PLAN": "3,0"}),
        ffma("warp_groups_2", g3, 1, {"SMMC_FORCE_PLAN": "1,1,2"}),
        ffma("warp_groups_4_last_arriver", g3, 1, {"SMMC_FORCE_PLAN": "1,3,4", "SMMC_CLUSTER_RED": "0"}),
        ffma("warp_groups_4_cluster", g3, 1, {"SMMC_FORCE_PLAN": "3,2,4", "SMMC_CLUSTER_RED": "1"}),
        ffma("warp_groups_reduce_kernel", g3, 1, {"SMMC_FORCE_PLAN": "1,8,2", "SMMC_CLUSTER_RED": "0"}),
        ffma("inkernel_split_S9_groups4", g3, 1, {"SMMC_FORCE_PLAN": "4,9,4,5"}),
        ffma("inkernel_split_S18_7x7", G(128, 72, 7, 7, 3), 2, {"SMMC_FORCE_PLAN": "4,18,2,5"}),
        ffma("inkernel_split_128x64", g3, 2, {"SMMC_FORCE_PLAN": "1,4,1,5"}),
        ffma("narrow_tile_128x32", G(64, 32, 20, 20, 3), 3, {"SMMC_FORCE_PLAN": "5,1"}),
        ffma("narrow_tile_last_arriver", G(32, 88, 17, 23, 5), 2, {"SMMC_FORCE_PLAN": "5,3", "SMMC_CLUSTER_RED": "0"}),
        ffma("narrow_tile_inkernel", G(64, 32, 20, 20, 3), 2, {"SMMC_FORCE_PLAN": "5,4,1,5"}),
        ffma("generic_order_ci3", G(3, 16, 12, 12, 5), 2, {"SMMC_STEM": "0"}),
        ffma("ragged_co37", G(24, 37, 11, 9, 3), 3, {}),
        ffma("planner_default_n1", G(128, 128, 14, 14, 3), 1, {}),
        ffma("stem_3x3s1", G(3, 64, 20, 20, 3), 2, {}),
        ffma("stem_3x3s1_round1", G(3, 64, 20, 20, 3), 2, {"SMMC_STEM_RW0": "1"}),
        ffma("stem_3x3s1_rw_tail", G(3, 40, 12, 24, 3), 3, {}),
        ffma("stem_3x3s1_rw_vgg", G(3, 64, 224, 224, 3), 1, {}),
        ffma("stem_3x3s1_scalar", G(3, 64, 18, 18, 3), 1, {"SMMC_STEM_SCALAR": "1"}),
        ffma("stem_7x7s2", G(3, 64, 30, 30, 7, 2, 3), 2, {}),
        ffma("stem_11x11s4", G(3, 96, 43, 43, 11, 4, 0), 2, {}),
        # narrow planes: a right-edge window's overhang spans rows (must not pass the tensor end)
        ffma("stem_11x11s4_narrow", ConvGeometry(3, 33, 13, 11, 11, 11, 4, 4, 0, 0), 2, {}),
        ffma("stem_7x7s2_narrow", ConvGeometry(2, 8, 9, 8, 7, 7, 2, 2, 3, 0), 3, {}),
        ffma("conv1x1_persistent", G(64, 64, 12, 12, 1, 1, 0), 2, {}),
        ffma("conv1x1_persistent_co128", G(32, 128, 8, 8, 1, 1, 0), 3, {}),
        ffma("conv1x1_tiled", G(64, 64, 12, 12, 1, 1, 0), 2, {"SMMC_1X1": "0"}),
        ffma("conv1x1_streamed_weights", G(64, 256, 12, 12, 1, 1, 0), 2, {"SMMC_1X1_WRES": "0"}),
        ffma("conv1x1_resident_w_co256", G(64, 256, 12, 12, 1, 1, 0), 3, {}),
        ffma("conv1x1_resident_w_co64", G(256, 64, 12, 12, 1, 1, 0), 2, {}),
        ffma("conv1x1_warp_tile", G(128, 64, 18, 18, 1, 1, 0), 15, {}),
        ffma("conv1x1_warp_tile_forced_ragged_co48", G(64, 48, 6, 6, 1, 1, 0), 3, {"SMMC_1X1_NARROW": "2"}),
        ffma("conv1x1_warp_tile_forced_multi_tile_warps", G(64, 64, 56, 56, 1, 1, 0), 12,
             {"SMMC_1X1_NARROW": "2"}),
        ffma("exact_mode", G(5, 7, 9, 8, 3), 2, {}, mode="exact", tol=0.0),
        # the planner's own N=1 plans of config 2 (tuning table: warp groups,
        # cluster DSMEM and reduce-kernel split-K)
        ffma("n1_cfg2_64@56", G(64, 64, 56, 56, 3), 1, {}),
        ffma("n1_cfg2_128@28", G(128, 128, 28, 28, 3), 1, {}),
        ffma("n1_cfg2_256@14", G(256, 256, 14, 14, 3), 1, {}),
        ffma("n1_cfg2_512@7", G(512, 512, 7, 7, 3), 1, {}),
    ]
    tc_cases = [
        ("tc_halo_nonpersistent", G(64, 128, 12, 12, 3), 2, {"SMMC_TC_PERSIST": "0"}),
        ("tc_halo_persistent_mt1", G(64, 128, 12, 12, 3), 2, {"SMMC_TC_PERSIST": "1", "SMMC_TC_MT": "1"}),
        ("tc_halo_persistent_mt2", G(64, 128, 12, 12, 3), 4, {"SMMC_TC_PERSIST": "1", "SMMC_TC_MT": "2"}),
        ("tc_halo_persistent_n256", G(64, 256, 8, 8, 3), 4, {"SMMC_TC_PERSIST": "1", "SMMC_TC_BN": "256"}),
        ("tc_box", G(64, 64, 10, 10, 3), 2, {"SMMC_TC_KERNEL": "b"}),
        ("tc_split", G(256, 64, 7, 7, 3), 1, {"SMMC_TC_SPLIT": "4"}),
        ("tc_1x1", G(64, 256, 8, 8, 1, 1, 0), 2, {}),
    ]
    hooks = ("SMMC_FORCE_PLAN", "SMMC_CLUSTER_RED", "SMMC_STEM", "SMMC_STEM_SCALAR", "SMMC_STEM_RW0", "SMMC_1X1",
             "SMMC_1X1_WRES",
             "SMMC_TC_PERSIST", "SMMC_TC_MT", "SMMC_TC_BN", "SMMC_TC_KERNEL", "SMMC_TC_SPLIT")

    def set_env(env):
        for k in hooks:
            os.environ.pop(k, None)
        os.environ.update(env)

    failures = 0
    seed = 1
    noise_stream = torch.cuda.Stream() if args.noise else None
    noise_a = torch.randn(2048, 2048, device="cuda") if args.noise else None

    def noise():
        if noise_stream is not None:
            with torch.cuda.stream(noise_stream):
                for _ in range(4):
                    noise_a.copy_(noise_a @ noise_a * 1e-3)

    for name, _, g, n, env, mode, tol in cases:
        if args.only and args.only not in name:
            continue
        set_env(env)
        seed += 1
        x, w = synthetic_layer(g, n, seed)
        ws = repack_weights(w, g)
        y = device.conv2d(torch.from_numpy(x).cuda(), torch.from_numpy(ws).cuda(), g, mode=mode)
        torch.cuda.synchronize()
        ref = orc.smm_conv_c(x, ws, g, threads=2)
        err = orc.max_abs_ratio(y.cpu().numpy(), ref)
        ok = (err == 0.0) if tol == 0.0 else err <= tol
        mism = 0
        if args.repeat > 1:
            xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(ws).cuda()
            out = torch.empty_like(y)
            for _ in range(args.repeat - 1):
                out.fill_(float("nan"))
                noise()
                device.conv2d(xd, wd, g, mode=mode, out=out)
                mism += not torch.equal(out, y)
            torch.cuda.synchronize()
            ok = ok and mism == 0
        failures += not ok
        print(f"{name:32s} {'ok' if ok else 'FAIL'} err={err:.2e}"
              + (f" relaunch mismatches {mism}/{args.repeat - 1}" if args.repeat > 1 else "")
              + f" plan: {_native.plan_describe(g, n, mode)}", flush=True)
    for name, g, n, env in tc_cases:
        if args.only and args.only not in name:
            continue
        set_env(env)
        seed += 1
        x, w = synthetic_layer(g, n, seed)
        layer = device.TcSmmConv2d(g, w)
        y = layer(layer.pack_input(torch.from_numpy(x).cuda()))
        torch.cuda.synchronize()
        ref = orc.smm_conv_c(x, repack_weights(w, g), g, threads=2)
        err = orc.max_abs_ratio(y.cpu().numpy(), ref)
        ok = err <= 2e-2
        failures += not ok
        print(f"{name:32s} {'ok' if ok else 'FAIL'} err={err:.2e} plan: "
              f"{_native.tc_plan_describe(g, n)}", flush=True)
    set_env({})
    if not args.only or "tc3" in args.only:
        g = G(32, 64, 9, 9, 3)
        x, w = synthetic_layer(g, 2, 99)
        layer = device.Tc3SmmConv2d(g, w)
        y = layer(torch.from_numpy(x).cuda())
        torch.cuda.synchronize()
        err = orc.max_abs_ratio(y.cpu().numpy(), orc.smm_conv_c(x, repack_weights(w, g), g))
        ok = err <= 1e-4
        failures += not ok
        print(f"{'tc3_split_bf16':32s} {'ok' if ok else 'FAIL'} err={err:.2e}", flush=True)
    if not args.only or "gather" in args.only:
        g = G(32, 40, 9, 9, 3)
        x, w = synthetic_layer(g, 2, 7)
        ws = repack_weights(w, g)
        xd = torch.from_numpy(x).cuda()
        outs = [torch.full((2,) + g.output_shape, float("nan"), device="cuda") for _ in range(3)]
        for r in range(3):
            lo, hi = cout_shard(g.out_channels, r, 3)
            device.conv2d_gather(xd, torch.from_numpy(np.ascontiguousarray(ws[..., lo:hi])).cuda(),
                                 outs, cout_geometry(g, lo, hi), lo, g.out_channels)
        torch.cuda.synchronize()
        ref = orc.smm_conv_c(x, ws, g)
        err = max(orc.max_abs_ratio(o.cpu().numpy(), ref) for o in outs)
        ok = err <= 1e-4
        failures += not ok
        print(f"{'gather_placement_3_replicas':32s} {'ok' if ok else 'FAIL'} err={err:.2e}", flush=True)
    if not args.only or "helpers" in args.only:
        import paper_2411_15659_b200 as smm
        g = G(3, 4, 7, 9, 3, 2, 1)
        x = smm.random_tensor(g.input_shape, 3)
        buf = np.zeros((g.padded_h, g.out_w), np.float32)
        smm.extract_slice(x, g, 1, 2, buf)
        dst = np.ones((5, 6), np.float32)
        smm.scalar_matrix_fma(np.float32(0.5), np.full((5, 6), 2.0, np.float32), dst)
        ok = bool(np.all(dst == 2.0))
        y = smm.smm_conv_single(x, smm.repack_weights(smm.random_tensor(g.weights_shape, 4), g), g)
        ok = ok and np.isfinite(y).all()
        failures += not ok
        print(f"{'helpers_host_entries':32s} {'ok' if ok else 'FAIL'}", flush=True)
    print(f"sanitize_cases: {failures} failures", flush=True)
    return 1 if failures else 0


if __name__ == "__main__":
    sys.exit(main())
