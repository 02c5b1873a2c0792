"""Summarise one final measurement set (tools/final_profile.sh outputs in gpurun_out/) into
profiles/<tag>_*: the bench lines, the ncu launch list, per-kernel ncu metrics of the full capture,
and profiles/score_kernel_traffic.json (DRAM bytes per launch of score_tc2_kernel)."""
import csv
import json
import os
import shutil
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r2_final"
G = "gpurun_out"
P = "profiles"
os.makedirs(P, exist_ok=True)
for src, dst in [("final_bench.json", f"{tag}_bench.json"), ("final_ref.json", f"{tag}_reference_bench.json"),
                 ("final_launches.csv", f"{tag}_launches.csv")]:
    if os.path.exists(os.path.join(G, src)):
        shutil.copy(os.path.join(G, src), os.path.join(P, dst))

bench = json.loads(open(os.path.join(G, "final_bench.json")).read().strip().splitlines()[-1])
ref = json.loads(open(os.path.join(G, "final_ref.json")).read().strip().splitlines()[-1])

# launch list: per-kernel totals and shares
rows = [r for r in csv.reader(open(os.path.join(G, "final_launches.csv"))) if len(r) > 10]
hdr = rows[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = r[ik].split("(")[0].replace("void ", "").split("<")[0].replace("as::", "")
    v = float(r[iv].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    v = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
    tot[name] += v
    cnt[name] += 1
allt = sum(tot.values())

# full capture: metrics per kernel
raw = list(csv.reader(open(os.path.join(G, "final_raw.csv"))))
rh, ru = raw[0], raw[1]
want = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.max.pct_of_peak_sustained_active",
        "smsp__issue_active.min.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
kern = {}
for r in raw[2:]:
    name = r[rh.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].replace("as::", "")
    kern[name] = {w: (r[rh.index(w)] + " " + ru[rh.index(w)]).strip() for w in want if w in rh}

def num(s):
    return float(s.split()[0].replace(",", ""))

tr = kern.get("score_tc2_kernel", {})
traffic = None
if tr:
    def to_bytes(s):
        v, u = s.split()[0], s.split()[1] if len(s.split()) > 1 else "byte"
        f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return float(v.replace(",", "")) * f
    traffic = to_bytes(tr["dram__bytes_read.sum"]) + to_bytes(tr["dram__bytes_write.sum"])
    json.dump({"kernel": "score_tc2_kernel", "dram_bytes_per_launch": traffic,
               "source": f"profiles/{tag}_profile.md (ncu --set full, one bench step = one launch)"},
              open(os.path.join(P, "score_kernel_traffic.json"), "w"), indent=1)

r = bench["roofline"]
L = []
L.append(f"# {tag}: C4 bench step (10^8 sampled candidates, M = 256, EI, k = 32), 1 x B200\n")
L.append("Commands: `tools/final_profile.sh` (one gpurun call): bench line, reference arm, ncu launch list of "
         "`bench.py --steps 2 --warmup 1 --no-cpu-baseline`, one `ncu --set full --clock-control none "
         "--import-source on -k regex:\"score_tc2|gen_kernel\" -c 2` capture (one bench step).\n")
L.append("## Bench line (device-timed, L2 flushed before each step)\n")
L.append("| | value |\n|---|---|")
L.append(f"| step | {bench['ms_per_step']:.3f} ms -> {bench['value']:.3e} candidates/s ({bench['valid_per_s']:.3e} valid/s); "
         f"SM clock {bench['clocks']['sm_mhz']} MHz, reasons {bench['clocks']['reasons']} |")
L.append(f"| score_tc2_kernel | {r['kernel_ms']:.3f} ms ({100 * r['kernel_share']:.1f} % of the step) |")
L.append(f"| gen_kernel | {r['gen']['ms']:.3f} ms ({100 * r['gen']['share']:.1f} %) |")
L.append(f"| roofline ({r['bound']}, {r['unit']}) | achieved {r['achieved']:.1f} / peak {r['peak']:.1f} = **{r['frac']:.3f}** |")
L.append(f"| e2e (C ABI, host buffers) | {bench['e2e']['ms_per_step']:.3f} ms -> {bench['e2e']['value']:.3e} candidates/s |")
cb = bench.get("cpu_baseline", {})
if cb:
    L.append(f"| CPU oracle, {cb['cores']} cores ({cb.get('cpu_model')}) | {cb['value']:.3e} candidates/s; one core "
             f"{cb['one_core']['value']:.3e} |")
L.append(f"| reference arm (all-core oracle) | {ref['value']:.3e} candidates/s |")
L.append("\n## Launch list (ncu, cold, serialised; 2 timed + 1 warm-up steps + e2e steps)\n")
L.append("| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    L.append(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / allt:.1f} % |")
L.append("\n## ncu --set full (one bench step)\n")
names = ["gen_kernel", "score_tc2_kernel"]
L.append("| metric | " + " | ".join(names) + " |\n|---|" + "---|" * len(names))
for w in want:
    L.append(f"| {w} | " + " | ".join(kern.get(n, {}).get(w, "") for n in names) + " |")
if traffic is not None:
    L.append(f"\nscore_tc2_kernel DRAM traffic per launch: {traffic / 1e9:.3f} GB (the compact list, 40 B per valid "
             f"candidate, read once; the tables and the fit are L2-resident).")
open(os.path.join(P, f"{tag}_profile.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L))
