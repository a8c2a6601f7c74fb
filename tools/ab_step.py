"""Median m-order dense chain step (CUDA events) for the librd build named by RD_LIB (A/B of
compile variants, tools/build_ab.sh; RD_VARIANT=d forces the DPX column count, RD_TMA /
RD_SPLIT_TAIL / RD_SPLIT_K / RD_TILE / RD_STREAM_K set rd_set_gemm_tma / rd_set_split_tail /
rd_set_split_k / rd_set_gemm_tile / rd_set_stream_k).
python tools/ab_step.py [m] [steps]"""
import os
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2409_17658_b200 as rd  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 9
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if os.environ.get("RD_VARIANT"):
    rd.rd_set_gemm_variant(int(os.environ["RD_VARIANT"]))
if os.environ.get("RD_TMA"):
    rd.rd_set_gemm_tma(int(os.environ["RD_TMA"]))
if os.environ.get("RD_SPLIT_TAIL"):
    rd.rd_set_split_tail(int(os.environ["RD_SPLIT_TAIL"]))
if os.environ.get("RD_SPLIT_K"):
    rd.rd_set_split_k(int(os.environ["RD_SPLIT_K"]))
if os.environ.get("RD_TILE"):
    rd.rd_set_gemm_tile(int(os.environ["RD_TILE"]))
if os.environ.get("RD_STREAM_K"):
    rd.rd_set_stream_k(int(os.environ["RD_STREAM_K"]))
st = torch.cuda.current_stream()
ch = rd.Chain(m, alpha_max=10, stream=st)
for _ in range(5):
    ch.step()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
for a, b in ev:
    a.record(st); ch.step(); b.record(st)
torch.cuda.synchronize()
t = statistics.median(a.elapsed_time(b) for a, b in ev)
tag = " ".join(f"{k}={os.environ[k]}" for k in ("RD_VARIANT", "RD_TMA", "RD_SPLIT_TAIL", "RD_SPLIT_K", "RD_TILE", "RD_STREAM_K") if k in os.environ)
print(f"{os.path.basename(os.environ.get('RD_LIB', 'librd.so'))} {tag} m={m} d={ch.gemm_variant} step {t:.3f} ms "
      f"({float(ch.N) ** 3 / t / 1e9:.1f} T)", flush=True)
ch.close()
