import numpy as np, sys
raw = open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/dbg_timing.bin", "rb").read()
it, nb = np.frombuffer(raw[:8], np.int32)
t = np.frombuffer(raw[8:], np.uint64).reshape(it, nb, -1).astype(np.int64)
valid = (t[:, :, 0] > 0).all(axis=1)
t = t[valid]
base = t[:, :, 0].min(axis=1, keepdims=True)
start = t[:, :, 0] - base
work = t[:, :, 1] - t[:, :, 0]
rel = t[:, :, 2] - base
print("iters", len(t), "blocks", nb)
print("start skew (max-min) ns: mean %.0f p50 %.0f" % (start.max(1).mean(), np.median(start.max(1))))
print("work ns per block: mean %.0f, max-over-blocks mean %.0f p50 %.0f p90 %.0f" % (work.mean(), work.max(1).mean(), np.median(work.max(1)), np.percentile(work.max(1), 90)))
arr = t[:, :, 1] - base
print("last work end ns (from first start): mean %.0f" % arr.max(1).mean())
print("release after last work end ns: mean %.0f p50 %.0f" % ((rel.min(1) - arr.max(1)).mean(), np.median(rel.min(1) - arr.max(1))))
print("release spread ns: mean %.0f" % (rel.max(1) - rel.min(1)).mean())
nxt = t[1:, :, 0] - t[:-1, :, 2]
print("release -> next start ns per block: mean %.0f p90 %.0f" % (nxt.mean(), np.percentile(nxt, 90)))
per = (t[1:, :, 0].min(1) - t[:-1, :, 0].min(1))
print("iteration period ns: mean %.0f p50 %.0f" % (per.mean(), np.median(per)))
slow = np.argmax(work, axis=1)
print("slowest block histogram (top):", np.bincount(slow, minlength=nb).argsort()[::-1][:8], np.sort(np.bincount(slow, minlength=nb))[::-1][:8])

# per-stage latencies of thread 0's first task (where recorded)
st = t[:, :, 3:7]
ok = (st > 0).all(axis=2)
if ok.any():
    d = np.diff(st, axis=2)[ok] / 1.965
    print("task stages ns (entry->record, record->dist, dist->candidates): mean",
          d.mean(0).round(0), "p90", np.percentile(d, 90, axis=0).round(0))
    loop = (t[:, :, 7] - t[:, :, 3])[ok] / 1.965
    print("thread-0 task loop from first task entry ns: mean %.0f p90 %.0f" % (loop.mean(), np.percentile(loop, 90)))
bp = t[:, :, 8:12]
okb = (bp > 0).all(axis=2)
if okb.any():
    d = np.diff(bp, axis=2)[okb] / 1.965
    print("barrier3 ns (release fence, poll wait, slot reduce): mean", d.mean(0).round(0),
          "p90", np.percentile(d, 90, axis=0).round(0))
# v4: end of publish (slot 8, globaltimer) relative to release (slot 2)
pb = t[:, :, 8]
okp = (pb > 0) & (pb >= t[:, :, 2]) & (pb - t[:, :, 2] < 100000)
if okp.any() and not okb.any():
    print("v4 post+publish ns: mean %.0f p90 %.0f" % ((pb - t[:, :, 2])[okp].mean(),
          np.percentile((pb - t[:, :, 2])[okp], 90)))
# v4: slowest warp of each CTA (slot 9) vs warp 0 (slot 10): cycles << 8 | flags
sw = t[:, :, 9]
w0 = t[:, :, 10]
if (sw > 0).any():
    cyc_s = (sw >> 8) / 1.965
    fl = sw & 0xff
    print("slowest warp loop ns: mean %.0f p90 %.0f; warp0 mean %.0f" % (cyc_s[sw > 0].mean(),
          np.percentile(cyc_s[sw > 0], 90), ((w0 >> 8) / 1.965)[w0 > 0].mean()))
    for name, bit in (("new-topleset task", 1), ("freeze", 2)):
        print("  slowest warp had %s: %.0f%%" % (name, 100 * ((fl[sw > 0] & bit) > 0).mean()))
    print("  slowest warp passes: ", np.bincount((fl[sw > 0] >> 3))[:6])
if (sw > 0).any():
    print("  slowest warp had fresh task: %.0f%%" % (100 * ((fl[sw > 0] & 4) > 0).mean()))
if t.shape[2] >= 16:
    k2 = t[:, :, 11:15].astype(np.float64)
    ok2 = t[:, :, 13] > 0
    if ok2.any():
        print("kind-2 first task (ns from entry): pv %.0f (spins mean %.2f, max %d) row %.0f cas %.0f" % (
            k2[..., 0][ok2].mean() / 1.965, k2[..., 1][ok2].mean(), k2[..., 1][ok2].max(),
            k2[..., 2][ok2].mean() / 1.965, k2[..., 3][ok2].mean() / 1.965))
# v4: stages of the CTA's first newest-topleset task (cycles; slots 9-15)
if t.shape[2] >= 16:
    kd = t[:, :, 9:16].astype(np.float64) / 1.965
    ok = (t[:, :, 9] > 0) & (t[:, :, 12] > 0)
    if ok.any():
        m = kd[ok].mean(0)
        print("first new-topleset task (ns): entry@%.0f  pv +%.0f  row +%.0f  dist +%.0f  candidates +%.0f  cas +%.0f  loop-end@%.0f" % (
            m[1], m[2], m[3], m[4], m[5], m[6], m[0]))
        if t.shape[2] >= 17:
            r = t[:, :, 16][ok].astype(np.float64) / 1.965
            print("   relax4 returned @%.0f (from iteration start)" % r.mean())
# wide iterations (slot 18 = 1): newest topleset (4-lane groups) vs older positions
# (one vertex per thread) vs barrier, globaltimer ns
if t.shape[2] >= 19:
    w = t[:, :, 18] == 1
    wi = w.all(axis=1)
    if wi.any():
        tw = t[wi]
        newest = (tw[:, :, 17] - tw[:, :, 0])
        older = (tw[:, :, 1] - tw[:, :, 17])
        bar = (tw[:, :, 2] - tw[:, :, 1])
        per = tw[:, :, 2].max(1) - tw[:, :, 0].min(1)
        print("wide iterations %d: newest-topleset part mean %.0f (max-over-CTAs %.0f), "
              "older part mean %.0f (max %.0f), barrier mean %.0f, start->last release %.0f ns" % (
                  wi.sum(), newest.mean(), newest.max(1).mean(), older.mean(), older.max(1).mean(),
                  bar.mean(), per.mean()))
