"""Build kernel-v3 experiment libraries lib<name>.so (A/B via SRHT_LIB; scripts/gpu_ab_v3.sh)."""
import concurrent.futures as cf
import json
import sys

sys.path.insert(0, '.')
from paper_0812_4547_b200 import build as b

V = json.loads(sys.argv[1])  # {"name": ["DEFINE=1", ...], ...}
with cf.ThreadPoolExecutor(len(V)) as ex:
    for name, out in zip(V, ex.map(lambda kv: b.build_variant(kv[0], kv[1]), V.items())):
        print(name, out)
