"""world_size-2/3 gloo check of the row-sharded dictionary join
(tsd.join_dictionary_sharded: block-aligned shard ranges from the C ABI's
tsd_dict_shard_rows, one all-gather), spawned by test_cpu.py. The per-shard
join is the oracle (no GPU here); the assembled profile must equal the
unsharded oracle join bit for bit, because shards are whole 16384-window
reference blocks (dictionary.hpp:175-180)."""
import os
import sys

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def worker(rank, world):
    os.environ["RANK"], os.environ["WORLD_SIZE"] = str(rank), str(world)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_12965_b200 as tsd
    from oracle import py_oracle as O
    from paper_2112_12965_b200 import synth
    m = 30
    q = synth.walk(11, 3 * 16384 + 5000)  # 4 reference blocks, the last one ragged
    segs = list(synth.walks(12, 3, 200))
    starts = [0, 200, 400]
    D = tsd.Dictionary([tsd.Segment(s, v) for s, v in zip(starts, segs)], m=m, source_length=600)
    P = tsd.join_dictionary_sharded(q, D, m, _shard_join=lambda x: O.dict_join(x, segs, starts, m))
    rv, ri = O.dict_join(q, segs, starts, m)
    assert P.values.shape == rv.shape and np.array_equal(P.indices, ri) and np.array_equal(P.values, rv)
    lo, hi = tsd.dict_shard_rows(q.size, m, rank, world)
    assert lo % 16384 == 0 and (hi % 16384 == 0 or hi == q.size - m + 1)
    if rank == 0:
        print("SHARD_OK", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(int(sys.argv[1]) if len(sys.argv) > 1 else 2,), nprocs=int(sys.argv[1]) if len(sys.argv) > 1 else 2,
             join=True)
