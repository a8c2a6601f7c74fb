"""Host-side overheads of a chain at small orders: create, one step + sync, destroy (wall clock)."""
import ctypes
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

torch.cuda.init()
L = rd.lib()
st = torch.cuda.Stream()
stats = torch.empty(41, dtype=torch.int32, device="cuda")
for m in [int(x) for x in sys.argv[1:]] or [3, 5, 7]:
    for method in (0, 1):
        tc, ts, td = [], [], []
        for _ in range(6):
            h = ctypes.c_void_p()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            assert L.rd_chain_create_ex(m, 10, 0, rd.count_words(m), method, ctypes.c_void_p(st.cuda_stream),
                                        ctypes.byref(h)) == 0
            t1 = time.perf_counter()
            L.rd_chain_step(h, ctypes.c_void_p(stats.data_ptr()))
            st.synchronize()
            t2 = time.perf_counter()
            L.rd_chain_destroy(h)
            t3 = time.perf_counter()
            tc.append(t1 - t0); ts.append(t2 - t1); td.append(t3 - t2)
        f = lambda v: f"{sorted(v)[len(v)//2]*1e3:.3f}"
        print(f"m={m} method={method} create {f(tc)} ms  step+sync {f(ts)} ms  destroy {f(td)} ms", flush=True)
