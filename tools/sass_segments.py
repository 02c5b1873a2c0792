"""Split an ncu `--page source --csv --print-source sass` dump at barrier / mbarrier-wait
instructions and sum warp-state samples and executed instructions per segment (dev aid)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) >= len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot_s = sum(int(r[ix["# Samples"]] or 0) for r in data)
seg = []
cur = {"start": data[0][0][-5:], "s": 0, "i": 0, "st": {}, "n": 0}
for r in data:
    s = int(r[ix["# Samples"]] or 0)
    n = int(r[ix["Instructions Executed"]] or 0)
    cur["s"] += s
    cur["i"] += n
    cur["n"] += 1
    for h in stalls:
        cur["st"][h] = cur["st"].get(h, 0) + int(r[ix[h]] or 0)
    src = r[1]
    if "BAR.SYNC" in src or "BAR.ARV" in src or "EXIT" in src:
        cur["end"] = r[0][-5:] + " " + src.strip()[:40]
        seg.append(cur)
        cur = {"start": r[0][-5:], "s": 0, "i": 0, "st": {}, "n": 0}
cur["end"] = "end"
seg.append(cur)
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
for c in seg:
    if c["s"] * 100.0 / tot_s < thr:
        continue
    top = sorted(c["st"].items(), key=lambda x: -x[1])[:3]
    print(f'{c["start"]}..{c["end"]:48s} n={c["n"]:5d} samples {c["s"]*100.0/tot_s:5.1f}% inst {c["i"]/1e6:9.1f}M  ' +
          " ".join(f"{k[6:]}:{v*100.0/max(1,c['s']):.0f}%" for k, v in top))
