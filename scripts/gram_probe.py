"""Gram of a config-4-shaped sketch (8192 x 513) or config-2-shaped batch (3000 x 101 x 1024) for
profiling: python scripts/gram_probe.py [4|2] [reps]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_0812_4547_b200 as srht  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
g = torch.Generator(device="cuda").manual_seed(0)
SM = (torch.randn((513, 8192), device="cuda", generator=g).t() if cfg == 4
      else torch.randn((3000, 101, 1024), device="cuda", generator=g))
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    G = srht.gram(SM)
    b.record()
    torch.cuda.synchronize()
    print("gram config", cfg, "ms", a.elapsed_time(b))
