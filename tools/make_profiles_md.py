#!/usr/bin/env python
"""Assemble profiles/round2.md from one tools/profile_final.sh run (gpurun_out/<T>_*).

  python tools/make_profiles_md.py r2f > profiles/round2.md
Copies the launch lists and bench lines it cites into profiles/ as well."""
import json
import os
import shutil
import subprocess
import sys

T = sys.argv[1] if len(sys.argv) > 1 else "r2f"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GO = os.path.join(ROOT, "gpurun_out")
PR = os.path.join(ROOT, "profiles")


def bench(cfg):
    p = os.path.join(GO, "bench_%s_%s.json" % (T, cfg))
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p))
    except Exception:
        return None


def summary(kind, *args):
    return subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), kind] + list(args),
                          capture_output=True, text=True).stdout


print("# Round 2 profiles (B200, final round-2 build)\n")
print("All numbers from `tools/profile_final.sh %s` on one B200 (clocks and throttle reasons are in every bench" % T)
print("line). Launch lists: `ncu --metrics gpu__time_duration.sum --clock-control none` of")
print("`bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-d1` (4 identical steps; cold-cache and")
print("serialised under ncu, so shares matter, not absolutes -- in the real step the vertex order runs beside the")
print("3D gradient and D0 beside D_{d-1}). Full captures: `ncu --set full --import-source on --clock-control none`.\n")
print("## 1. Bench lines (`bench.py`, device time, inputs resident; e2e = host field in, diagrams out)\n")
print("| Config | M vertices/s | ms/step | e2e M vertices/s | order | gradient | critical | D0 | D_{d-1} | D1 pairs / generators (s) | roofline.frac (gradient kernel, HBM) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for cfg in ("c4", "c3", "c5a", "c5b", "c2", "c1", "c4_5tet", "c3_5tet"):
    d = bench(cfg)
    if not d:
        continue
    s = d["stages_ms_per_step"]
    d1 = d.get("d1")
    d1s = "%.3f / %.3f (%d pairs)" % (d1["ms_pairs"] / 1e3, d1["ms_generators"] / 1e3, d1["pairs"]) if d1 else "—"
    print("| %s | %.0f | %.2f | %s | %.2f | %.2f | %.2f | %.2f | %.2f | %s | %.4f |" % (
        cfg.replace("_5tet", " (five tetrahedra)"), d["value"], d["ms_per_step"],
        "%.0f" % d["e2e"]["value"] if d.get("e2e") else "—", s["order"], s["gradient"], s["critical"], s["d0"],
        s["dtop"], d1s, d["roofline"]["frac"]))
    shutil.copy(os.path.join(GO, "bench_%s_%s.json" % (T, cfg)), os.path.join(PR, "bench_%s_%s.json" % (T, cfg)))
print("\nStage times overlap (order beside the gradient on a second stream, D0 beside D_{d-1}).\n")
ref = os.path.join(GO, "bench_%s_reference.json" % T)
if os.path.exists(ref):
    for line in open(ref):
        if line.startswith("{"):
            r = json.loads(line)
            print("`bench.py --impl reference` (the CPU oracle, %s): %.4f %s, %.1f ms per step.\n" % (
                r["cpu_baseline"]["sample"], r["value"], r["unit"], r["ms_per_step"]))
print("## 2. Launch lists (share of one step's device time)\n")
for cfg in ("c4", "c3", "c5a", "c5b"):
    p = os.path.join(GO, "%s_launches_%s.csv" % (T, cfg))
    if os.path.exists(p):
        shutil.copy(p, os.path.join(PR, "%s_launches_%s.csv" % (T, cfg)))
        print("### %s\n" % cfg)
        out = summary("launches", p, "4").splitlines()
        print("\n".join(out[:14] + out[-2:]))
        print()
print("## 3. `--set full` captures\n")
for name in ("k_gradient_pool3_c4", "k_os_pass_c4", "k_uf_coop_c5b", "k_d1_bigc_c4_256"):
    p = os.path.join(GO, "%s_%s.ncu-rep" % (T, name))
    if os.path.exists(p):
        print("### %s\n" % name)
        print(summary("full", p))
