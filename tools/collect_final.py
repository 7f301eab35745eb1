"""Copy the outputs of tools/job_r2_final.sh (gpurun_out/z.*) into profiles/ (round-2 names)."""
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PRO = os.path.join(ROOT, "profiles")


def last_json(path):
    line = None
    for l in open(path, errors="replace"):
        l = l.strip()
        if l.startswith("{") and l.endswith("}"):
            line = l
    return line


def put_json(src, dst):
    p = os.path.join(OUT, src)
    if not os.path.exists(p):
        print("missing", src)
        return None
    l = last_json(p)
    if l is None:
        print("no json line in", src)
        return None
    open(os.path.join(PRO, dst), "w").write(l + "\n")
    d = json.loads(l)
    print(dst, d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"))
    return d


def trim_details(src, dst, header, keep):
    p = os.path.join(OUT, src)
    if not os.path.exists(p):
        print("missing", src)
        return
    txt = open(p, errors="replace").read()
    parts = re.split(r"(?m)^(?=  void )", txt)
    out = [header] + [parts[1 + i].rstrip() for i in keep if 1 + i < len(parts)]
    open(os.path.join(PRO, dst), "w").write("\n".join(out) + "\n")
    print(dst, len(parts) - 1, "kernels, kept", keep)


put_json("z.bench_c2.log", "r2_bench_c2.json")
put_json("z.bench_c1.log", "r2_bench_c1.json")
put_json("z.bench_2d_L9.log", "r2_bench_2d_L9.json")
put_json("z.bench_2d_L10.log", "r2_bench_2d_L10.json")
put_json("z.ref.c2.log", "r2_bench_reference_c2.json")
put_json("z.ref.c1.log", "r2_bench_reference_c1.json")
put_json("z.ref.2d.log", "r2_bench_reference_2d.json")
for src, dst in (("z.c2_bench_launches.csv", "r2_c2_bench_launches"), ("z.2d_L9_bench_launches.csv", "r2_2d_bench_launches"),
                 ("z.2d_L10_bench_launches.csv", "r2_2d_L10_bench_launches")):
    p = os.path.join(OUT, src)
    if not os.path.exists(p):
        print("missing", src)
        continue
    shutil.copy(p, os.path.join(PRO, dst + ".csv"))
    s = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "launch_summary.py"), p], capture_output=True, text=True)
    open(os.path.join(PRO, dst + "_summary.txt"), "w").write(s.stdout)
    print(dst, s.stdout.splitlines()[1:4])
trim_details("z_flow_c2.details.txt", "r2_c2_flow_leg_ncu_full.txt",
             "# ncu --set full --import-source on --clock-control none -k regex:k_flow_leg -s 2 -c 2 python tools/flow_once.py c2 "
             "(c2 level-0 dataflow smoothing legs, down then up; tools/job_r2_final.sh)", [0, 1])
trim_details("z_tri_c2.details.txt", "r2_c2_tri_tma_ncu_full.txt",
             "# ncu --profile-from-start off -k regex:k_tri_tma -c 2 --set full --import-source on --clock-control none "
             "python tools/apply_p_once.py (the forward and backward factor sweeps of one prolongation on config 2; "
             "tools/job_r2_final.sh)", [0, 1])
