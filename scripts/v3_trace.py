"""Per-phase timing of kernel v3 on CTA 0 (clock64 at phase boundaries; experiment only).

python scripts/v3_trace.py [n d r]  (default: config-4 shape 2^20 x 513, r = 8192)
Group g producer warp 0 (tiles f = g, g+2, ...) and consumer thread 0: medians over flat tiles 16..79,
then the whole traced run (tiles 0..4095) to show where the mean departs from the median."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht
from paper_0812_4547_b200 import _lib

n, d, r = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (1 << 20, 512, 8192))]
c = d + 1
M = torch.empty((c, n), dtype=torch.float32, device="cuda").t()
srht.gen_uniform(0, 0, M)
plan = srht.Plan(n, d, r, 0)
ws = plan.workspace(c)
out = torch.empty((c, r), device="cuda").t()
lib = _lib.load()
T = 4096
tr = torch.zeros(3 * T * 8, dtype=torch.int64, device="cuda")
lib.srht_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
for _ in range(3):
    plan.sketch_columns(M, out=out, workspace=ws)
torch.cuda.synchronize()
lib.srht_debug_set_trace(ctypes.c_void_p(0))
print("kernel:", lib.srht_debug_last_kernel(), "shape", n, d, r)
tt = tr.cpu().numpy().reshape(3, T, 8).astype(np.float64)
np.save('gpurun_out/v3_trace_raw.npy', tt) if len(sys.argv) > 4 else None
t = tt[:, 16:80]
order = [0, 6, 1, 2, 3, 4, 5]
pn = ["TMA wait", "R1 LDS+signs+quarters", "R1 stage 12", "bar1+stage 13+STS", "bar2+R2 LDS+stages", "R2 last stage+STS+arrive"]
for g in range(2):
    rows = t[g, g::2][:30]
    rows = rows[rows[:, 0] > 0]
    print("producer group %d: tile-to-tile %.0f cycles (median, own tiles)" % (g, np.median(np.diff(rows[:, 0]))))
    for k in range(6):
        print("   %-26s %7.0f" % (pn[k], np.median(rows[:, order[k + 1]] - rows[:, order[k]])))
    print("   %-26s %7.0f" % ("to next tile", np.median(rows[1:, 0] - rows[:-1, 5])))
rows = t[2][t[2][:, 0] > 0]
print("consumer t0: tile-to-tile %.0f" % np.median(np.diff(rows[:, 0])))
for k, nm in enumerate(["READY wait+1st LDTM", "gather", "refill (last warp only)"]):
    print("   %-22s %7.0f" % (nm, np.median(rows[:, k + 1] - rows[:, k])))
# cross-role: when does the producer finish tile f vs consumer start it
fin = {f: t[f % 2, f - 16, 5] for f in range(16, 80) if t[f % 2, f - 16, 5] > 0}

# ---- whole traced run: mean vs median, slow tiles and where they fall ----
for g in range(2):
    st = tt[g, g::2, 0]
    st = st[st > 0]
    dt = np.diff(st)
    print("group %d, %d tiles: tile-to-tile mean %.0f median %.0f p90 %.0f p99 %.0f max %.0f; time in >2x-median gaps %.1f%%"
          % (g, len(st), dt.mean(), np.median(dt), np.percentile(dt, 90), np.percentile(dt, 99), dt.max(),
             100 * dt[dt > 2 * np.median(dt)].sum() / dt.sum()))
    w = tt[g, g::2]
    w = w[w[:, 0] > 0]
    wait = w[:, 6] - w[:, 0]
    print("   TMA wait mean %.0f median %.0f p90 %.0f" % (wait.mean(), np.median(wait), np.percentile(wait, 90)))
    nxt = w[1:, 0] - w[:-1, 5]
    print("   to next tile mean %.0f median %.0f p90 %.0f" % (nxt.mean(), np.median(nxt), np.percentile(nxt, 90)))
    slow = np.argsort(dt)[-8:]
    print("   slowest gaps (flat tile, cycles):", [(int(2 * i + g), int(dt[i])) for i in sorted(slow)])
cs = tt[2, :, 0]
cs = cs[cs > 0]
print("consumer t0, %d tiles: tile-to-tile mean %.0f median %.0f; span %.0f cycles" % (len(cs), np.diff(cs).mean(), np.median(np.diff(cs)), cs[-1] - cs[0]))
ep = tt[2][(tt[2][:, 4] > 0)]
if len(ep):
    e = ep[:, 5] - ep[:, 4]
    print("consumer slab epilogue (%d items): mean %.0f median %.0f max %.0f" % (len(e), e.mean(), np.median(e), e.max()))
# TMA latency: refill issue (consumer trace slot 6, indexed by the loaded tile) to the
# producer's FULL wait completing (producer slot 6); when the producer did not wait only
# the lead (issue -> producer starts waiting) is known
iss = tt[2, :, 6]
lat, lead = [], []
for f in range(3, T):
    g = f % 2
    if iss[f] > 0 and tt[g, f, 6] > 0 and tt[g, f, 0] > 0:
        lead.append(tt[g, f, 0] - iss[f])
        if tt[g, f, 6] - tt[g, f, 0] > 300:
            lat.append(tt[g, f, 6] - iss[f])
if lead:
    print("refill lead (issue -> producer starts waiting): median %.0f p10 %.0f p90 %.0f" % (np.median(lead), np.percentile(lead, 10), np.percentile(lead, 90)))
if lat:
    print("refill latency when the producer waited (%d of %d tiles): median %.0f p10 %.0f p90 %.0f" % (len(lat), len(lead), np.median(lat), np.percentile(lat, 10), np.percentile(lat, 90)))
