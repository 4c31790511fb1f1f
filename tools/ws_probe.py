"""Probe of the warp-specialised attend: one small case through wildcat_attend with WC_ATTEND=ws vs the
default tcgen05 path on the same cache.  usage: python tools/ws_probe.py [m] [r] [d] [heads]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc  # noqa: E402
from paper_2602_10056_b200.inputs import make_qkv  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 256
r = int(sys.argv[2]) if len(sys.argv) > 2 else 128
d = int(sys.argv[3]) if len(sys.argv) > 3 else 128
h = int(sys.argv[4]) if len(sys.argv) > 4 else 1
dev = torch.device("cuda:0")
Q, K, V = (x.to(dev) for x in make_qkv(1, h, 1, m, max(4 * r, 1024), d, "bf16", "G", 0))
sel = wc.select(Q, K, r, seed=0, block=16)
cache = wc.weights(K, V, sel)
O_ref = wc.attend(Q, cache)
torch.cuda.synchronize()
os.environ["WC_ATTEND"] = "ws"
print("running ws ...", flush=True)
O_ws = wc.attend(Q, cache)
torch.cuda.synchronize()
err = (O_ws.float() - O_ref.float()).abs().max().item()
print(f"m={m} r={r} d={d} h={h}: max |ws - tc| = {err:.3e}", flush=True)
