"""Per-block phase trace of the blocked selection at the headline (run with WC_SELECT_TRACE=1).
usage: python tools/trace_blocked.py [block]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc  # noqa: E402
from paper_2602_10056_b200.inputs import make_qkv  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 16
Q, K, V = make_qkv(1, 1, 1, 65536, 65536, 128, "bf16", "G", 0)
dev = torch.device("cuda:0")
sel = wc.select(Q.to(dev), K.to(dev), 256, seed=0, block=b)
torch.cuda.synchronize()
print("stats", sel.stats[0, :10].tolist(), file=sys.stderr, flush=True)
