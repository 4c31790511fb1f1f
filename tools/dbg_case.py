import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from wc_harness import compare, qkv
args = sys.argv[1:]
b, hq, hkv, m, n, d, r = map(int, args[:7]); dt = args[7]; fam = args[8] if len(args) > 8 else "G"
Q, K, V = qkv(b, hq, hkv, m, n, d, dt, fam, seed=0)
out = compare(Q, K, V, r, dt)
print("err", out["err"])
