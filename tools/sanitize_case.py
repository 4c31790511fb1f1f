"""One small WildCat call per case, for compute-sanitizer runs (memcheck / racecheck / synccheck).
usage: python tools/sanitize_case.py CASE   (cfg1 | vit | blocked | binned | kv | decode | nshard_p2p)"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc  # noqa: E402
from paper_2602_10056_b200.inputs import make_qkv  # noqa: E402

case = sys.argv[1]
dev = torch.device("cuda:0")


def dv(*ts):
    return [t.to(dev) for t in ts]


if case == "cfg1":  # BASELINE configs[0], sequential and blocked
    Q, K, V = dv(*make_qkv(1, 1, 1, 256, 256, 16, "f32", "G", 0))
    wc.forward(Q, K, V, 16, seed=0)
    wc.forward(Q, K, V, 16, seed=0, block=16)
elif case == "vit":  # ViT shape on 4 batches (48 units): SMEM-resident selection, tcgen05 weights/attend
    Q, K, V = dv(*make_qkv(4, 12, 12, 197, 197, 64, "bf16", "C", 0))
    wc.forward(Q, K, V, 32, seed=0, block=16)
    wc.forward(Q, K, V, 32, seed=0, block=1)
elif case == "blocked":  # one unit, n = 16K, r = 96: multi-CTA blocked selection (grid barrier, PDL,
    # bulk-copy ring), tcgen05 weights and attend, split solve
    Q, K, V = dv(*make_qkv(1, 1, 1, 4096, 16384, 128, "bf16", "G", 0))
    wc.forward(Q, K, V, 96, seed=0, block=16)
    wc.forward(Q, K, V, 96, seed=0, block=1)
elif case == "longr":  # r = 320 > 256: the streamed attend and the multi-panel solve
    Q, K, V = dv(*make_qkv(1, 2, 1, 1000, 3000, 128, "bf16", "G", 0))
    wc.forward(Q, K, V, 320, seed=0, block=16)
elif case == "binned":
    Q, K, V = dv(*make_qkv(2, 4, 2, 512, 4096, 64, "bf16", "G", 0))
    wc.forward(Q, K, V, 64, seed=0, block=8, bins=8)
elif case == "kv":  # KV-cache compression + decode
    Q, K, V = dv(*make_qkv(1, 8, 2, 64, 4096, 128, "bf16", "L", 0))
    cache = wc.compress_kv(Q, K, V, 96, keep_first=32, keep_last=32, bins=8, block=16)
    Qd = dv(*make_qkv(1, 8, 2, 1, 16, 128, "bf16", "L", 1))[0]
    wc.attend(Qd, cache)
elif case == "finite":
    Q, K, V = dv(*make_qkv(1, 2, 1, 33, 301, 64, "bf16", "G", 1))
    wc.forward(Q, K, V, 16, seed=1, check_finite=True)
else:
    raise SystemExit(f"unknown case {case}")
torch.cuda.synchronize()
print(f"{case}: ok")
