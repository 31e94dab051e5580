"""Build A/B libraries that differ only in the stem kernel thread tiles
(lib/ab/<name>.so; conv_stem.cu recompiled with SV*_ defines, linked with the
main build objects).  Run from the repo root after the main build."""
import subprocess, sys
sys_path_fix = __import__("sys").path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from pathlib import Path
from paper_2411_15659_b200 import build as b
V = {
 "m3a": ("SV3", (4,16,2,256,1,22,1,3)), "m3b": ("SV3", (4,16,2,256,1,23,1,3)), "m3c": ("SV3", (4,16,2,128,2,22,1,3)),
 "m3d": ("SV3", (4,16,2,384,1,22,1,3)), "m3e": ("SV3", (4,16,2,128,3,22,1,3)), "m3f": ("SV3", (4,16,2,192,1,22,1,3)),
 "m3g": ("SV3", (4,16,2,320,1,22,1,3)), "m3h": ("SV3", (4,16,4,256,1,22,1,3)),
}
exe = b.nvcc()
objs = [str(o) for o in sorted(Path("build/smmc").glob("*.o")) if o.stem != "conv_stem"]
procs = []
for k, (pre, (px, cpt, ng, t, mb, pf, *gg)) in V.items():
    ci = gg[1] if len(gg) > 1 else 0
    d = [f"-D{pre}_PX={px}", f"-D{pre}_CPT={cpt}", f"-D{pre}_NG={ng}", f"-D{pre}_T={t}",
         f"-D{pre}_MINB={mb}", f"-D{pre}_PF={int(pf)}", f"-D{pre}_G={gg[0] if gg else 1}", f"-D{pre}_CI={ci}"]
    if pre == "SV1": d.append("-DSTEM_K1=1")
    obj = f"/tmp/stem_{k}.o"
    cmd = [exe, *b.ARCH, *b.NVCC_FLAGS, *d, "-c", "paper_2411_15659_b200/csrc/conv_stem.cu", "-o", obj]
    procs.append((k, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
for k, obj, p in procs:
    out, _ = p.communicate()
    assert p.returncode == 0, out.decode()[-3000:]
    spill = [l for l in out.decode().splitlines() if "spill" in l and not l.strip().startswith("0 bytes stack frame, 0 bytes spill stores")]
    lib = f"paper_2411_15659_b200/lib/ab/{k}.so"
    Path(lib).parent.mkdir(parents=True, exist_ok=True)
    subprocess.run([exe, *b.ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", lib, obj, *objs,
                    "-lcudart_static", "-lrt", "-ldl", "-lpthread", "-Xlinker", "--no-undefined"], check=True)
    print(k, "spills:", spill)
