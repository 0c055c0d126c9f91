"""C4 end-to-end probe (development tool): tsd_dict_join with pinned host
buffers, TSD_VERBOSE phases. usage: TSD_VERBOSE=1 python tools/e2eprobe.py [reps]"""
import sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import bench
import paper_2112_12965_b200 as tsd
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
D, segs = bench.make_dictionary()
q = bench.make_query(4)
nrows = q.size - bench.M + 1
h_q = torch.from_numpy(q).pin_memory()
h_val = torch.empty(nrows, dtype=torch.float64).pin_memory()
h_idx = torch.empty(nrows, dtype=torch.int64).pin_memory()
seg_all = np.ascontiguousarray(np.concatenate(list(segs)))
lib = tsd.load_library()
lens = np.full(bench.N_SEG, bench.SEG_LEN, dtype=np.uintp)
starts = np.arange(bench.N_SEG, dtype=np.uintp) * bench.SEG_LEN
f64p, i64p, szp = ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_size_t)
for r in range(reps + 1):
    t0 = time.perf_counter()
    rc = lib.tsd_dict_join(ctypes.cast(h_q.data_ptr(), f64p), bench.Q_LEN, seg_all.ctypes.data_as(f64p),
                           lens.ctypes.data_as(szp), starts.ctypes.data_as(szp), bench.N_SEG, bench.M, 0,
                           ctypes.cast(h_val.data_ptr(), f64p), ctypes.cast(h_idx.data_ptr(), i64p))
    assert rc == 0, lib.tsd_last_error()
    print(f"call {r}: {(time.perf_counter() - t0) * 1e3:.1f} ms", file=sys.stderr, flush=True)
