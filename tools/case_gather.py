import sys, os, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2602_10056_b200 as wc
from wc_harness import qkv
Q, K, V = qkv(1, 2, 2, 50, 5000, 64, "bf16", "G", seed=21)
dev = torch.device("cuda:0")
s1 = wc.select(Q.to(dev), K.to(dev), 100, seed=21, block=int(sys.argv[1]))
torch.cuda.synchronize(); print("ok", s1.S[0, :8].tolist())
