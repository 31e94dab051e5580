"""Print a compact table of gpurun_out/bench_cfg*.json (bench.py --details)."""
import glob
import json
import sys

pats = sys.argv[1:] or ["gpurun_out/bench_cfg*.json"]
for f in [f for p in pats for f in sorted(glob.glob(p))]:
    j = json.load(open(f))
    cpu = j.get("cpu_baseline") or {}
    print(f"{f}: value={j['value']} GFLOP/s ms/step={j['ms_per_step']} e2e={j['e2e']['value'] if j.get('e2e') else None} "
          f"cpu={cpu.get('value')} clocks={j['clocks']['sm_mhz']} {j['clocks']['reasons']} "
          f"parity={cpu.get('gpu_vs_oracle_max_err_ratio', float('nan')):.2e} launches={j['gpu_launches']}")
    for L in j["layers"]:
        print(f"   {L['layer']:30s} {L['ms_avg'] * 1e3:9.1f}us {L['tflops']:7.2f} TF {L['frac_fp32_peak']:.3f}  {L['plan'][6:]}")
