"""Quick device timing of one power step (GEMM + fused stats) per m, CUDA events."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2409_17658_b200 as rd  # noqa: E402

import os
ms = [int(x) for x in sys.argv[1:]] or [7, 8, 9]
variants = [int(v) for v in os.environ.get("VARIANTS", "3").split(",")]
method = int(os.environ.get("METHOD", "0"))
rd.rd_set_sparse_variant(int(os.environ.get("SPV", "3")))
for v, m in [(v, m) for v in variants for m in ms]:
    rd.rd_set_gemm_variant(v)
    t0 = time.time()
    ch = rd.Chain(m, alpha_max=10, stream=torch.cuda.current_stream(), method=method)
    torch.cuda.synchronize()
    tb = time.time() - t0
    N = ch.N
    for _ in range(3):
        ch.step()
    torch.cuda.synchronize()
    reps = 10 if m <= 8 else 4
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ch.step()
    e1.record()
    torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / reps * 1e-3
    terms = ch.terms_per_step
    print(f"method={method} variant={v} m={m} N={N} build={tb:.2f}s step={dt*1e3:.3f} ms  "
          f"{terms/dt/1e12:.3f} T terms/s  dense-equivalent {N**3/dt/1e12:.2f} T/s", flush=True)
    ch.close()
print(rd.rd_alu_probe())
