"""Summarise a round's ncu captures into profiles/<round>/ (tracked)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

src = sys.argv[1]          # gpurun_out/r01
dst = sys.argv[2]          # profiles/r01
os.makedirs(dst, exist_ok=True)

# ---- launch lists: per-kernel time share (serialised launches: compare SHARES) and DRAM traffic per launch
def launch_table(fname, title):
    rows = list(csv.reader(open(os.path.join(src, fname))))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ix = {k: i for i, k in enumerate(hdr)}
    agg = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    for r in data:
        k = r[ix["Kernel Name"]].split("(")[0]
        m, u, v = r[ix["Metric Name"]], r[ix["Metric Unit"]], float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        agg[k][m] += v * scale
        if m == "gpu__time_duration.sum":
            cnt[k] += 1
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    lines = [title, "", "| kernel | launches | total us | avg us | share | DRAM read+write per launch (MB) |",
             "|---|---|---|---|---|---|"]
    traffic = {}
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        n = cnt[k]
        rw = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / max(n, 1)
        lines.append(f"| {k} | {n} | {a['gpu__time_duration.sum']:.1f} | {a['gpu__time_duration.sum']/n:.2f} | "
                     f"{a['gpu__time_duration.sum']/tot:.3f} | {rw/1e6:.2f} |")
        traffic[k] = rw
    return lines, traffic


common = ("C3 shapes (8192 envs, n = 100, 3x512, T = 256 rollouts + GAE + fitness + selection; --cache-control none: "
          "L2 warm across launches, so DRAM write-backs of one launch land in the next ones and the per-launch "
          "average over the window counts reads and writes)")
lines, traffic = launch_table("launches_c3.csv", "# ncu launch list, headline path (fused rollout kernel): " + common)
if os.path.exists(os.path.join(src, "launches_c3_sep.csv")):
    l2, t2 = launch_table("launches_c3_sep.csv", "# ncu launch list, separate actor / env-step launches "
                          "(POD_FUSED=0, the C5 path): " + common)
    lines += [""] + l2
    for k, v in t2.items():   # the separate kernels' traffic from the path that runs them every step
        if "actor_forward" in k or "env_step" in k or k not in traffic:
            traffic[k] = v
open(os.path.join(dst, "ncu_launches_c3.md"), "w").write("\n".join(lines) + "\n")

# ---- one --set full capture per hot kernel
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum"]
summ = {}
out = ["# ncu --set full captures (one launch each, C3 shapes, T = 256: the fused rollout kernel runs all 256 steps "
       "in its one launch; actor_forward / env_step from the POD_FUSED=0 path)", ""]
for k in ("rollout_fused", "actor_forward", "env_step", "gae"):
    rep = os.path.join(src, f"prof_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    hh, uu, vv = r[0], r[1], r[2]
    d = {}
    for a, u, v in zip(hh, uu, vv):
        if a in want:
            d[a] = f"{v} {u}".strip()
    summ[k] = d
    out.append(f"## {k}")
    out += [f"- {a}: {d[a]}" for a in want if a in d]
    out.append("")
open(os.path.join(dst, "ncu_full_summary.md"), "w").write("\n".join(out) + "\n")

# ---- per-launch DRAM traffic of the hot kernels, for bench.py's roofline.traffic: the multi-launch window of
# the launch list (read + write, averaged over the launches of each kernel)
names = {"pod::actor_forward_kernel": "actor_mlp", "gae": "gae"}
tj = {}
for k, rw in traffic.items():
    if "rollout_fused" in k:
        tj["rollout_fused"] = rw
    elif "actor_forward" in k:
        tj["actor_mlp"] = rw
    elif "env_step_kernel" in k:
        tj["env_step"] = max(tj.get("env_step", 0.0), rw)
    elif "gae" in k and "normalize" not in k:
        tj["gae"] = max(tj.get("gae", 0.0), rw)
json.dump({"C3": tj, "_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch, averaged over the launches of a "
           "T = 256 C3 rollout with the L2 warm between launches (ncu --cache-control none; profiles/"
           + os.path.basename(dst) + "/ncu_launches_c3.md)"},
          open(os.path.join(os.path.dirname(dst), "ncu_traffic.json"), "w"), indent=1)
print("\n".join(lines))
print("\n".join(out))
