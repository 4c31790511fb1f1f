"""Worker for tests/test_gpu_nshard.py::test_p2p_two_ranks_one_gpu (test infrastructure only).

Launched as `python tests/nshard_p2p_worker.py <rank> <world> <port> <out.npz>` by the test: every
rank runs on cuda:0 (the test box has one GPU), bootstraps a gloo group on 127.0.0.1, builds the
device-initiated (p2p) communicator -- CUDA-IPC-mapped mailboxes, handles all-gathered over gloo --
and runs wildcat_forward_nshard on its contiguous key shard; rank 0 saves S, r_eff and its output."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2602_10056_b200 as wc  # noqa: E402
from paper_2602_10056_b200.inputs import make_qkv  # noqa: E402


def main():
    rank, world, port, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
    n, m, d, r, seed = int(os.environ.get("WC_T_N", 8192)), 256, 64, 24, 7
    block = int(os.environ.get("WC_T_BLOCK", 1))
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    dev = torch.device("cuda:0")
    Q, K, V = make_qkv(1, 2, 1, m, n, d, "bf16", "G", seed=3)
    off, cnt = wc.shard_range(n, world, rank)
    comm = wc.NshardComm.create(world, rank, transport="p2p", capacity=max(r * (d + 1), 16 * (2 + d + r)) + 64)
    S = torch.empty(r, dtype=torch.int32, device=dev)
    R = torch.empty(1, dtype=torch.int32, device=dev)
    Kl, Vl = K[:, :, off:off + cnt].to(dev), V[:, :, off:off + cnt].to(dev)
    O = wc.forward_nshard(comm, Q.to(dev), Kl, Vl, r, n, off, seed=seed, S=S, r_eff=R, block=block)
    torch.cuda.synchronize()
    if rank == 0:
        np.savez(out, S=S.cpu().numpy(), r_eff=R.cpu().numpy(), O=O.float().cpu().numpy())
    dist.barrier()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
