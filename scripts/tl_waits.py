"""Per-role wait totals from a timeline captured with PB_TC_PROF=1 (record type 4:
warp, elapsed, waits on w_empty, b_full, a_full, w_full, a_empty in ns), medians over CTAs."""
import sys
import numpy as np
rec = np.load(sys.argv[1])
r4 = rec[rec[:, 0] == 4]
tl = rec[rec[:, 0] == 1]
print("CTAs", int(tl[:, 1].max()) + 1, "calls", len(tl) // (int(tl[:, 1].max()) + 1))
names = ["w_empty", "b_full", "a_full", "w_full", "a_empty"]
for w in sorted(set(r4[:, 2].tolist())):
    sel = r4[r4[:, 2] == w]
    print(f"warp {w:2d}: elapsed {np.median(sel[:,3])/1e3:7.2f} us  " +
          "  ".join(f"{n} {np.median(sel[:,4+i])/1e3:6.2f}" for i, n in enumerate(names)))
t0 = tl[:, 4].min()
for name, col in (("start", 4), ("bready", 5), ("mma0", 6), ("mend", 7), ("cend", 8), ("end", 9)):
    v = (tl[:, col] - t0) / 1e3
    print(f"{name:6s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f}")
r3 = rec[rec[:, 0] == 3]
if len(r3):
    # per segment: {3, cta, seg, units, wake, drained, done, cycles wake->first ld, t ld done, cycles ld->drained}
    d = (r3[:, 5] - r3[:, 4]) / 1e3
    f = (r3[:, 6] - r3[:, 5]) / 1e3
    w = (r3[:, 4] - t0) / 1e3
    print(f"segments {len(r3)}: drain med {np.median(d):.2f} max {d.max():.2f} us; finalise med {np.median(f):.2f} "
          f"max {f.max():.2f} us; wake med {np.median(w):.2f}")
    for q in (50, 90, 99):
        print(f"  p{q}: drain {np.percentile(d, q):.2f} finalise {np.percentile(f, q):.2f}")
    l = (r3[:, 8] - r3[:, 4]) / 1e3
    print(f"  wake -> first TMEM load done: med {np.median(l):.2f} max {l.max():.2f} us; cycles {np.median(r3[:,7]):.0f}, "
          f"first load -> drained cycles {np.median(r3[:,9]):.0f}")
