"""Debug helper: run one forward at a large-r shape (no oracle)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import make_qkv

d, r = int(sys.argv[1]), int(sys.argv[2])
Q, K, V = (t.cuda() for t in make_qkv(1, 4, 2, 300, 3000, d, "bf16", "G", 11))
S = torch.empty(2, r, dtype=torch.int32, device="cuda")
R = torch.empty(2, dtype=torch.int32, device="cuda")
O = wc.forward(Q, K, V, r, seed=11, S=S, r_eff=R)
torch.cuda.synchronize()
print("ok", R.tolist(), O.float().abs().max().item())
