"""Debug: per-round phase timing of the selection kernel (CTA 0), WC_SELECT_TRACE=1."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2602_10056_b200 as wc
from paper_2602_10056_b200.inputs import CONFIGS, make_config

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "headline"]
Q, K, V = make_config(cfg)
dev = torch.device("cuda:0")
Qd, Kd, Vd = Q.to(dev), K.to(dev), V.to(dev)
wc.forward(Qd, Kd, Vd, cfg.r)
torch.cuda.synchronize()
