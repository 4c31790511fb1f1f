import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import make_qkv
Q, K, V = make_qkv(1, 1, 1, 65536, 65536, 128, "bf16", "G", 0)
dev = torch.device("cuda:0")
Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
print("env", os.environ.get("WC_SELECT_TRACE"), file=sys.stderr, flush=True)
for b in (16,):
    sel = wc.select(Qd, Kd, 256, seed=0, block=b)
    torch.cuda.synchronize()
    print("stats", sel.stats[0, :9].tolist(), file=sys.stderr, flush=True)
