"""Gram A/B (config 4 / config 2 shapes): per-call CUDA-event times plus a digest of G, so two
library builds (SRHT_LIB=...) can be checked bit-identical.  python scripts/gram_ab.py CFG REPS"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_0812_4547_b200 as srht  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = torch.Generator(device="cuda").manual_seed(0)
SM = (torch.randn((513, 8192), device="cuda", generator=g).t() if cfg == 4
      else torch.randn((3000, 101, 1024), device="cuda", generator=g))
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    G = srht.gram(SM)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ts = sorted(ts[3:])
dig = hashlib.sha256(G.cpu().numpy().tobytes()).hexdigest()[:16]
print("lib %s config %d median_ms %.4f min_ms %.4f digest %s" % (os.environ.get("SRHT_LIB", "libsrht.so"), cfg,
      ts[len(ts) // 2], ts[0], dig))
