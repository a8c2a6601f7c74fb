"""Dense m = 9 step time on torch's legacy stream vs a non-blocking stream vs the C loop."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

torch.cuda.init()
m, steps = 9, 8
for name, stream in (("legacy", None), ("nonblocking", torch.cuda.Stream()), ("legacy2", None)):
    with torch.cuda.stream(stream) if stream is not None else torch.cuda.stream(torch.cuda.default_stream()):
        ch = rd.Chain(m, alpha_max=10, stream=stream)
        ch.step().cpu()
        t0 = time.perf_counter()
        for _ in range(steps):
            ch.step().cpu()
        dt = (time.perf_counter() - t0) / steps
        ch.close()
    print(f"{name}: {dt*1e3:.1f} ms per step", flush=True)
for rep in range(2):
    r = rd.rd_power_sequence(m, 10, 10)     # 9 steps, no detection
    print(f"C loop kmax=10: chain {r['t_chain']*1e3/9:.1f} ms per step", flush=True)
