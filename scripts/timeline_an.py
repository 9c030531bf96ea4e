"""Summarise scripts/timeline.py records (include/pb.h pb_debug_timeline layout)."""
import sys
import numpy as np

rec = np.load(sys.argv[1])
ta = rec[rec[:, 0] == 0]
tl = rec[rec[:, 0] == 1]
t0 = min(ta[:, 4].min() if len(ta) else 1 << 62, tl[:, 4].min())
f = lambda v: (v - t0) / 1000.0
ncta = int(tl[:, 1].max()) + 1
nact = int(ta[:, 1].max()) + 1 if len(ta) else 0
tl = tl[np.argsort(tl[:, 4], kind="stable")]
ta = ta[np.argsort(ta[:, 4], kind="stable")]
calls = len(tl) // ncta
for c in range(calls):
    g = tl[c * ncta:(c + 1) * ncta]
    print(f"call {c}:")
    if nact:
        a = ta[c * nact:(c + 1) * nact]
        print(f"  act  launch {f(a[:,4].min()):8.2f}..{f(a[:,4].max()):8.2f}  go {f(a[:,5].min()):8.2f}..{f(a[:,5].max()):8.2f}"
              f"  end {f(a[:,6].min()):8.2f}..{f(a[:,6].max()):8.2f}")
    for name, col in (("start", 4), ("bready", 5), ("mma0", 6), ("mend", 7), ("cend", 8), ("end", 9)):
        v = f(g[:, col])
        print(f"  gemm {name:6s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f}")
    u = g[:, 3]
    for uu in sorted(set(u.tolist())):
        sel = u == uu
        print(f"    units {uu}: n={sel.sum()} mma0->mend med {np.median((g[sel,7]-g[sel,6])/1000):.2f} us, "
              f"cend med {np.median(f(g[sel,8])):.2f}, end med {np.median(f(g[sel,9])):.2f}")
    late = g[f(g[:, 4]) > f(g[:, 4]).min() + 5]
    if len(late):
        print(f"  late-starting CTAs: {len(late)} on SMs {sorted(late[:,2].tolist())[:20]}")
pr = rec[rec[:, 0] == 2]
if len(pr):
    pr = pr[np.argsort(pr[:, 4], kind="stable")]
    for c in range(len(pr) // ncta):
        q = pr[c * ncta:(c + 1) * ncta]
        print(f"prologue call {c}: pdl-wait done {f(q[:,4]).min():8.2f}..{f(q[:,4]).max():8.2f}  "
              f"max done {f(q[:,5]).min():8.2f}..{f(q[:,5]).max():8.2f}  chunk0 done {f(q[:,6]).min():8.2f}..{f(q[:,6]).max():8.2f}  "
              f"slice done {f(q[:,7]).min():8.2f}..{f(q[:,7]).max():8.2f}")
        if q[:, 8].any():
            print(f"   max->f_b med {np.median(q[:,8]-q[:,5])/1e3:.2f}  f_b->groups done med {np.median(q[:,9]-q[:,8])/1e3:.2f}"
                  f"  groups->chunk0 published med {np.median(q[:,6]-q[:,9])/1e3:.2f} us; chunk groups: ballot loop "
                  f"med {np.median(q[:,2]):.0f} cycles, stores med {np.median(q[:,3]):.0f} cycles")
ep = rec[rec[:, 0] == 3]
if len(ep):
    # per epilogue segment: d_full wake -> TMEM drained -> slot/atomic done -> y stored
    last = ep[ep[:, 4] > np.median(tl[:, 9]) - 40000] if False else ep
    d1 = (ep[:, 5] - ep[:, 4]) / 1e3
    d2 = (ep[:, 6] - ep[:, 5]) / 1e3
    d3 = (ep[:, 7] - ep[:, 6]) / 1e3
    if ep[:, 8].any():
        dl = (ep[:, 8] - ep[:, 4]) / 1e3
        print(f"epilogue: wake -> TMEM loads done med {np.median(dl):.2f} max {dl.max():.2f} us; cycles: loads med "
              f"{np.median(ep[:,7]):.0f}, math+release med {np.median(ep[:,9]):.0f} max {ep[:,9].max():.0f}")
    print(f"epilogue segments {len(ep)}: TMEM->s_tot med {np.median(d1):.2f} max {d1.max():.2f} us; "
          f"slot+atomic med {np.median(d2):.2f} max {d2.max():.2f}; final med {np.median(d3):.2f} max {d3.max():.2f}")
    for kind, name in ((1, "whole"), (2, "finalizer"), (0, "parker")):
        sel = ep[:, 3] == kind
        if sel.any():
            tot = (ep[sel, 7] - ep[sel, 4]) / 1e3
            print(f"   {name:9s} n={sel.sum():4d} total med {np.median(tot):.2f} max {tot.max():.2f} us")
    # last CTA end relative to d_full wake of the final segment in each CTA
    tlk = tl[np.argsort(tl[:, 4], kind="stable")]
    e_end = {}
    for r_ in ep:
        e_end.setdefault(int(r_[1]), []).append(r_)
pf = rec[rec[:, 0] == 4]
if len(pf):
    names = ["w_empty", "b_full", "a_full", "w_full", "a_empty"]
    for w in range(11):
        q = pf[pf[:, 2] == w]
        if not len(q):
            continue
        tot = np.median(q[:, 3]) / 1e3
        nm = names if w < 3 else ["convert", "st_wait"] + names[2:]
        if w == 1:
            nm = ["d_empty"] + names[1:]
        parts = "  ".join(f"{n} {np.median(q[:, 4 + i]) / 1e3:6.2f}" for i, n in enumerate(nm) if q[:, 4 + i].any())
        print(f"  warp {w:2d}: total {tot:6.2f} us  waits(med, us): {parts}")

fp = rec[rec[:, 0] == 5]
if len(fp):
    fp = fp[np.argsort(fp[:, 4], kind="stable")]
    for c in range(len(fp) // ncta):
        q = fp[c * ncta:(c + 1) * ncta]
        print(f"first pass (warp 3) call {c}: start {f(q[:,4]).min():8.2f}..{f(q[:,4]).max():8.2f}  tiles {f(q[:,5]).min():8.2f}..{f(q[:,5]).max():8.2f}"
              f"  converted {f(q[:,6]).min():8.2f}..{f(q[:,6]).max():8.2f}  published {f(q[:,7]).min():8.2f}..{f(q[:,7]).max():8.2f}"
              f"  chunk0 B {f(q[:,8]).min():8.2f}..{f(q[:,8]).max():8.2f}")
if len(fp):
    for c in range(len(fp) // ncta):
        q = fp[c * ncta:(c + 1) * ncta]
        print(f"chunk0 call {c}: x issued {f(q[:,2]).min():8.2f}..{f(q[:,2]).max():8.2f}  f ready {f(q[:,3]).min():8.2f}..{f(q[:,3]).max():8.2f}"
              f"  built {f(q[:,8]).min():8.2f}..{f(q[:,8]).max():8.2f}  (build med {np.median((q[:,8]-q[:,3])/1e3):.2f} us)")
t6 = rec[rec[:, 0] == 6]
if len(t6):
    t6 = t6[np.argsort(t6[:, 2], kind="stable")]
    for c in range(len(t6) // ncta):
        q = t6[c * ncta:(c + 1) * ncta]
        base = q[:, 2].max()                      # the last CTA's MMA end
        rel = lambda col: (q[:, col] - base) / 1e3
        print(f"tail call {c} (us after the LAST mend): mend spread {(q[:,2].max()-q[:,2].min())/1e3:.2f}; "
              f"last seg wake med {np.median(rel(3)):.2f} max {rel(3).max():.2f}; drained med {np.median(rel(4)):.2f} "
              f"max {rel(4).max():.2f}; added max {rel(5).max():.2f}; bar arrive max {rel(6).max():.2f}; "
              f"bar exit med {np.median(rel(7)):.2f} max {rel(7).max():.2f}; fin med {np.median(rel(8)):.2f} "
              f"max {rel(8).max():.2f}; end max {rel(9).max():.2f}")
