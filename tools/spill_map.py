"""Where a score_tc2 instance spills: STL/LDL counts per SETMAXREG region (dev aid).
python tools/spill_map.py LIB.so [kernel-substring]"""
import re, subprocess, sys
lib = sys.argv[1]
pat = sys.argv[2] if len(sys.argv) > 2 else "score_tc2_kernelILi16ELi0ELi2ELi16"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(out) if "Function :" in l and pat in l)
end = next((i for i in range(start + 1, len(out)) if "Function :" in out[i]), len(out))
region, counts, size = "setup", {}, {}
for l in out[start:end]:
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if not m:
        continue
    ins = m.group(2)
    if "SETMAXREG" in ins:
        region = "producers" if "ALLOC" in ins and "DEALLOC" not in ins else "aux"
    c = counts.setdefault(region, [0, 0])
    size[region] = size.get(region, 0) + 16
    if re.search(r"\bSTL\b", ins):
        c[0] += 1
    if re.search(r"\bLDL\b", ins):
        c[1] += 1
for r in counts:
    print(f"{r:10s} code {size[r]/1024:6.1f} KB  STL {counts[r][0]:4d}  LDL {counts[r][1]:4d}")
