"""Write the round's profiles/ files from one tools/gpu_final.sh pass.

  python tools/final_profiles.py r01v13 v13
reads gpurun_out/<TAG>_*, writes profiles/r01_{bench,bench_reference,configs,scaling,launches}_<V>.*
"""
import collections
import csv
import io
import json
import re
import sys

tag, ver = sys.argv[1], sys.argv[2]
G = f"gpurun_out/{tag}"


def line(path):
    return json.loads(open(path).read().strip().splitlines()[-1])


bench = line(f"{G}_bench.json")
json.dump(bench, open(f"profiles/r01_bench_{ver}.json", "w"), indent=1)
json.dump(line(f"{G}_bench_ref.json"), open(f"profiles/r01_bench_reference_{ver}.json", "w"), indent=1)

keys = ["value", "ms_per_step", "n_gpus", "config", "roofline", "e2e", "clocks", "gpu_launches"]
cfgs = {"note": "round-1 final pass (tools/gpu_final.sh) on one 4-GPU B200 box: every BASELINE.json config; "
                "device time max over ranks; e2e through the C ABI with pinned host copies (absent for C5 at N=1: "
                "--no-e2e, 1M-token host buffers); 8 GPUs not offered by gpurun",
        "c4_n1": {k: bench.get(k) for k in keys}}
for name in ["c1", "c2", "c3_n1", "c3_n2", "c3_n4", "c3_n4_2x2", "c4_n2", "c4_n4", "c4_n4_2x2", "c5_n1", "c5_n4",
             "c5_n4_2x2"]:
    d = line(f"{G}_cfg_{name}.json")
    cfgs[name] = {k: d.get(k) for k in keys}
json.dump(cfgs, open(f"profiles/r01_configs_{ver}.json", "w"), indent=1)

v1 = bench["value"]
scal = {"note": f"device tokens/s (max over ranks), one 4-GPU B200 box, profiles/r01_configs_{ver}.json; "
                "scaling strong (512K fixed)"}
for key, name in [("1", "c4_n1"), ("2", "c4_n2"), ("4", "c4_n4"), ("4_2x2", "c4_n4_2x2")]:
    c = cfgs[name]
    scal[key] = {"value": c["value"], "e2e": (c["e2e"] or {}).get("value"),
                 "phase_ms": c["roofline"]["phase_ms"], "vs_n1": c["value"] / v1}
json.dump(scal, open(f"profiles/r01_scaling_{ver}.json", "w"), indent=1)

# launch list: ncu csv -> per-kernel totals
txt = open(f"{G}_launches.csv").read()
txt = txt[txt.index('"ID"'):]
rows = list(csv.DictReader(io.StringIO(txt)))
tot, cnt, bwd = collections.OrderedDict(), collections.Counter(), []
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    ms = float(r["Metric Value"]) / (1e6 if r["Metric Unit"] == "ns" else 1e3 if r["Metric Unit"] == "us" else 1)
    name = re.sub(r"\(.*", "", r["Kernel Name"])[:120]
    tot[name] = tot.get(name, 0.0) + ms
    cnt[name] += 1
    if "attn_bwd_kernel" in name:
        bwd.append(round(ms, 1))
s = sum(tot.values())
steps = 4
own = sum(c for n, c in cnt.items() if not n.startswith(("cub::", "at::", "void cub", "void at"))) // steps
with open(f"profiles/r01_launches_{ver}.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none, command:\n"
            "# python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline  (4 hot-path steps at S=524288, "
            "Hq=16, Hkv=2, p=0.9)\n# cold-cache, serialised per-launch times; compare SHARES with bench phase_ms\n"
            f"# own kernels per step: {own} (cub / torch fill kernels excluded)\n# total_ms  launches  share  kernel\n")
    for n, t in sorted(tot.items(), key=lambda kv: -kv[1]):
        f.write(f"{t:10.2f} {cnt[n]:5d} {100 * t / s:6.2f}%  {n}\n")
    f.write(f"# sum {s:.2f} ms over {steps} steps = {s / steps:.1f} ms/step; attn_bwd launches (block, bar, ...) ms: "
            f"{bwd}\n# live bench (profiles/r01_bench_{ver}.json) phase_ms = {bench['roofline']['phase_ms']}\n")
print(open(f"profiles/r01_launches_{ver}.txt").read())
