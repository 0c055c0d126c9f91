"""world_size-2 gloo check of the sharded self-join's exchange step
(tsd.exchange_partials: all-gather + acc_merge via tsd_profile_merge),
spawned by test_cpu.py. Shard partials come from a long-double-free numpy
brute force (every pair once, both rows updated, pairs split by row parity),
so the test needs no GPU."""
import os
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def corr_matrix(t, m):
    W = np.lib.stride_tricks.sliding_window_view(t, m)
    Z = W - W.mean(1, keepdims=True)
    Z /= np.sqrt((Z * Z).sum(1, keepdims=True))
    return np.clip(Z @ Z.T, -1.0, 1.0)


def partial(C, excl, rank, world):
    cnt = C.shape[0]
    corr, col = np.full(cnt, -2.0), np.full(cnt, -1, dtype=np.int64)
    for i in range(rank, cnt, world):  # this shard's pairs: rows i = rank mod world
        for j in range(i + excl + 1, cnt):  # profiles.hpp:287-297 updates both rows
            for a, b in ((i, j), (j, i)):
                c = C[i, j]
                if col[a] < 0 or c > corr[a] or (c == corr[a] and b < col[a]):
                    corr[a], col[a] = c, b
    return corr, col


def worker(rank, world):
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_12965_b200 as tsd
    from paper_2112_12965_b200 import synth
    m, t = 16, synth.walk(31, 260)
    excl = m // 2
    C = corr_matrix(t, m)
    corr, col = tsd.exchange_partials(*partial(C, excl, rank, world))
    full_c, full_j = partial(C, excl, 0, 1)
    assert np.array_equal(col, full_j) and np.array_equal(corr, full_c)
    if rank == 0:
        print("SELFSHARD_OK", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2,), nprocs=2, join=True)
