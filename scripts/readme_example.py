"""The README's Python example, run as written (plus a KKT check of the NNLS solution)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_0812_4547_b200 as srht

n, d, r = 1 << 20, 512, 8192
A = torch.rand(d, n, device="cuda").t()          # column-major float32 (n, d)
b = torch.rand(n, device="cuda")
plan = srht.Plan(n, d, r, seed=0)                 # D and K (Philox), slot layouts; reusable
SA, Sb = plan.sketch(A, b)                        # (r, d), (r,)
G = srht.gram(torch.column_stack([SA, Sb]))       # FP64 [[SA'SA, SA'Sb], [Sb'SA, Sb'Sb]]
x, iters = srht.nnls_gram(G)                      # Algorithm 1 step 5: argmin_{x>=0} ||SA x - Sb||
Q, q = G[:d, :d], G[:d, d]
w = q - Q @ x                                     # dual: <= 0 off the support, ~0 on it
print("iters", int(iters), "support", int((x > 0).sum()), "max dual off-support %.3g" % float(w[x == 0].max()),
      "max |dual| on support %.3g" % float(w[x > 0].abs().max()), "scale", float(q.abs().max()))
