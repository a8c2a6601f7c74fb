import sys, torch
sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd
from paper_2409_17658_b200 import dist as D
for on in (False, True):
    rd.rd_set_split_k(on)
    for m, r0, r1 in ((6, 0, 848), (7, 0, 2507), (8, 0, 1024), (8, 0, 1920), (9, 0, 2816)):
        ch = rd.Chain(m, alpha_max=10, row_begin=r0, row_end=r1)
        for _ in range(3): ch.step()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): ch.step()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print("splitk", on, m, r1 - r0, round(ms, 3), "ms", round((r1 - r0) * ch.N ** 2 / ms / 1e9, 2), "T/s", flush=True)
        ch.close()
