"""Summarise the CTA-0 phase timeline written by score_tc2_kernel when AS_TC2_TRACE=<file> is set
(development aid).  Events (per tile t, lane 0 of every warp, clock64):
  producers: 0 loop top, 1 after publish(t+1), 2 after produce(t) rest, 3 after head of t+1,
             4 after d_full wait, 5 after D read + barrier, 6 after acquisition, 7 after admission
  MMA warp : 8 before d_empty wait, 9 after it, 11 chunk NA issued, 10 last commit of tile t
"""
import sys
import numpy as np

TILES, EV, W = 64, 16, 18
a = np.fromfile(sys.argv[1], dtype=np.uint64)
rec = TILES * EV * W
n = a.size // rec
x = a[(n - 1) * rec:n * rec].reshape(TILES, EV, W).astype(np.int64)
prod = x[:, :, :16]
mma = x[:, :, 16]
ok = [t for t in range(2, TILES - 1) if prod[t, 0].min() > 0 and prod[t + 1, 0].min() > 0]
print(f"{n} records, {len(ok)} steady tiles")
tile = np.array([np.median(prod[t + 1, 0] - prod[t, 0]) for t in ok])
print("tile period (median over warps) cycles: mean %.0f" % tile.mean())
names = ["publish", "produce rest", "head t+1", "wait d_full", "D read", "bar+finalize", "admit"]
for e in range(1, 8):
    d = np.array([prod[t, e] - prod[t, e - 1] for t in ok])          # [tiles, warps]
    print(f"  {names[e-1]:14s} mean over warps %7.0f  warp0-3 %7.0f  warp4-15 %7.0f  max %7.0f" %
          (d.mean(), d[:, :4].mean(), d[:, 4:].mean(), d.max(axis=1).mean()))
dm = np.array([mma[t, 9] - mma[t, 8] for t in ok])
print("  MMA d_empty wait %.0f" % dm.mean())
print("  MMA: d_empty-> chunk NA issued %.0f, -> last commit %.0f" %
      (np.mean([mma[t, 11] - mma[t, 9] for t in ok]), np.mean([mma[t, 10] - mma[t, 9] for t in ok])))
print("  d_full wait start (warp0) vs MMA last commit: %.0f" % np.mean([prod[t, 3, 0] - mma[t, 10] for t in ok]))
pe = [(5, 13, "finalize: sums"), (13, 14, "finalize: acq32"), (14, 6, "finalize: rest"), (6, 7, "finalize: admit")]
for a_, b_, nm in pe:
    d = np.array([prod[t, b_, :4] - prod[t, a_, :4] for t in ok])
    print(f"  {nm:18s} warps 0-3 mean %7.0f  max %7.0f" % (d.mean(), d.max(axis=1).mean()))
wa = np.array([x[t, 12, 16] for t in ok]); wb = np.array([x[t, 13, 16] for t in ok])
print("  MMA warp per tile: waiting a_full %.0f cycles, waiting b_full %.0f cycles" % (wa.mean(), wb.mean()))
r_t = np.array([x[t, 12, 17] for t in ok]); r_r = np.array([x[t, 13, 17] for t in ok]); r_x = np.array([x[t, 14, 17] for t in ok])
print("  R2 warp per tile: waiting t_ready %.0f, r_empty %.0f, x_full (T stage) %.0f cycles" % (r_t.mean(), r_r.mean(), r_x.mean()))
