#!/usr/bin/env python
"""Benchmark: the (min,+) power step of arXiv 2409.17658 on B200.

A "step" is one pass of the whole hot path over the m = 9 transfer matrix
(N = C_9 = 21909): A^k = A^{k-1} (x) A on the DPX GEMM with the fused diagonal min and
periodicity stats (a2-a4), the stats all_reduce(MIN) across ranks, the device->host read
of the stats and the host decision (a5).  The right operand A is packed once before the
timed region (a1).  One process per GPU; ranks own 128-row panels of the output.

    python bench.py [--gpus N --steps K --warmup W] [--order-m 9] [--form replicated|allgather|peer] [--impl reference]

Prints ONE JSON line on rank 0 (contract in DESIGN.md §Measurement).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_K80_GOPS = {6: 99.6, 7: 156.9, 8: 143.1, 9: 166.2}   # BASELINE.md §1.1 (derived from Table 3)
SM_COUNT = 148
NNZ = {1: 7, 2: 33, 3: 167, 4: 836, 5: 4195, 6: 21043, 7: 105566, 8: 529584, 9: 2656733, 10: 13327868}  # nnz A(G)
DPX_MINPLUS_PER_CLK_SM = 128      # VIADDMNMX.S16x2 at half rate: 64 lanes x 2 (measured)
# Unit-count bound of the (min,+) term over every instruction form the GEMM can use (DESIGN.md
# §5): alu and fma pipes 2 warp-instr/clk/SM each (rt_SMSP = 2, B300_MICROARCH "Pipe rates"),
# issue 4/clk/SM.  DPX VIADDMNMX.S16x2 = 2 terms on alu; IMAD packed add (fma) x2 + VIMNMX3
# (alu) = 4 terms.  Best mix 1 DPX : 1 (2 IMAD + VIMNMX3) per SMSP-pair slot -> 64 + 128 terms.
PIPE_MINPLUS_PER_CLK_SM = 192
SM_MAX_MHZ = 1965.0
# dram__bytes_read.sum + dram__bytes_write.sum per GEMM launch from `ncu --set full`
# (profiles/), by m; None where not captured for the current kernel
TRAFFIC = {9: 46845147720}   # profiles/r02p_gemm_ncu_summary.txt (TMA mainloop, d = 3, A^9): 45.862 GB read + 0.983 GB write


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--order-m", dest="m", type=int, default=9,
                   help="m of P_m (named to stay unambiguous next to torchrun's own options)")
    p.add_argument("--alpha-max", type=int, default=10)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--ttp-m", type=int, nargs="*", default=[3, 4, 5, 6, 7, 8, 9])
    p.add_argument("--oracle-ttp-m", type=int, nargs="*", default=[3, 4, 5, 6, 7, 8])
    p.add_argument("--gops-m", type=int, nargs="*", default=[3, 4, 5, 6, 7, 8])
    p.add_argument("--invariance-m", type=int, default=8, help="order of the operand-invariance check (0: off)")
    p.add_argument("--ttp-structured-only-m", type=int, nargs="*", default=[10])
    p.add_argument("--no-m11", action="store_true", help="skip the m = 11 structured chain run at >= 4 ranks")
    p.add_argument("--form", default="replicated", choices=["replicated", "allgather", "peer"],
                   help="replicated: A packed on every rank, row panels of A^(k-1) (x) A (default); "
                        "allgather: A^k = A (x) A^(k-1), A^(k-1) gathered over a P2P ring each step; "
                        "peer: A^k = A (x) A^(k-1) with the GEMM reading A^(k-1) from every rank's ring "
                        "(CUDA IPC / NVLink peer memory, the gather fused into the product)")
    return p.parse_args()


# ------------------------------------------------------------------- clocks --
class ClockSampler:
    """NVML SM clock + throttle reasons sampled every 100 ms while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, device_index: int):
        self.samples, self.power, self.reasons, self.max_mhz = [], [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons)}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w": round(statistics.median(self.power), 1) if self.power else None}


# -------------------------------------------------------------- CPU oracle --
class OracleSample:
    """The oracle's dense (min,+) loop (or_minplus_bt: i-j-k, guarded INF, OpenMP over the
    output) on sampled rows of the same step A^{k-1} (x) A(G): rows of a fully finite
    A^k-like operand (rd_inputs.power_like, seeded) times the real A(G) of m."""

    def __init__(self, m: int):
        import numpy as np

        import oracle as O
        O.build()
        self.O, self.m = O, m
        A = O.matrix(m)
        self.N = A.shape[0]
        self.BT = np.ascontiguousarray(A.T)

    def calibrate(self, seconds: float) -> int:
        from rd_inputs import power_like
        X = power_like(1, self.N, self.m, seed=0).astype("int32")
        t = time.perf_counter()
        self.O.minplus_bt(X, self.BT)
        return max(1, min(4096, int(seconds / max(time.perf_counter() - t, 1e-4))))

    def run(self, rows: int, seed: int = 1):
        """Returns (Gop/s, seconds) for `rows` output rows."""
        from rd_inputs import power_like
        X = power_like(rows, self.N, self.m, seed=seed).astype("int32")
        t = time.perf_counter()
        self.O.minplus_bt(X, self.BT)
        dt = time.perf_counter() - t
        return rows * self.N * self.N / dt / 1e9, dt


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _measured_hbm_gbs():
    """HBM copy bandwidth from MEASURED_PEAKS.json (driver-written), else the profiling guide's
    fallback of 6.5 TB/s."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6500.0


def cores_used():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


# ------------------------------------------------------------------- arms --
def run_reference(args, rank, world):
    """The oracle as it stands, on the host cores, on a bounded sample of the same
    workload (each step: a fixed number of sampled output rows); rank 0 only."""
    if rank != 0:
        return
    smp = OracleSample(args.m)
    N = smp.N
    rows = smp.calibrate(args.cpu_seconds / max(1, args.steps + args.warmup) * 3)
    times = []
    for i in range(args.warmup + args.steps):
        _, dt = smp.run(rows, seed=1 + i)
        if i >= args.warmup:
            times.append(dt)
    value = rows * N * N * len(times) / sum(times) / 1e9
    sample = f"{rows} sampled output rows of A^(k-1) (x) A(G) per step, m={args.m}, N={N}, dense i-j-k oracle"
    line = {
        "impl": "reference", "metric": "(min,+) Gop/s on A^(k-1) (x) A(G) at order N = C_m (power step with fused diag-min + periodicity test)",
        "value": round(value, 3), "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "i32",
        "data": "synthetic A^k-like rows (seeded) x deterministic A(G)",
        "config": {"workload": f"P_{args.m} box C_n: power step A^k = A^(k-1) (x) A(G), N = C_{args.m} = {N}",
                   "m": args.m, "N": N},
        "cpu_baseline": {"value": round(value, 3), "unit": "Gop/s", "cores": cores_used(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank, backend="nccl"):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2409_17658_b200 as rd
    from paper_2409_17658_b200 import dist as rdist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    m, am = args.m, args.alpha_max
    N = rd.count_words(m)
    r0, r1 = rdist.panel_bounds(N, world, rank)
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        if args.form == "peer":
            # fused all-gather: each rank's GEMM reads A^(k-1) from every rank's ring (CUDA IPC)
            chain = rdist.peer_chain(m, am, stream=stream)
            if world > 1:
                dist.barrier()
        elif world > 1 and args.form == "replicated":
            # A(G) built and packed once on rank 0, broadcast over NVLink (not rebuilt per rank)
            chain = rdist.broadcast_chain(m, am, r0, r1)
        else:
            chain = rd.Chain(m, alpha_max=am, row_begin=r0, row_end=r1, stream=stream) if r1 > r0 else None
        stats = torch.empty(rd.rd_stats_len(am), dtype=torch.int32, device=dev)
        neutral = torch.from_numpy(rdist.neutral_stats(am)).to(dev)
        hstats = torch.empty(rd.rd_stats_len(am), dtype=torch.int32, pin_memory=True)
    torch.cuda.synchronize()
    probe = rd.rd_alu_probe()          # live issue rates of the GEMM's instruction forms
    launches_per_step = 2 if chain is not None else 0   # stats init + GEMM (librd kernels)

    k_state = {"k": 1, "found": None}
    if args.form == "allgather":
        bounds = [rdist.panel_bounds(N, world, s) for s in range(world)]
        A_rows = torch.from_numpy(np.ascontiguousarray(rd.rd_build_matrix(m)[r0:r1])).to(dev)
        ag = {"ring": {1: A_rows.clone()}}
        if chain is not None:
            chain.close()
            chain = None
        launches_per_step = 3 * world + 3   # per ring chunk: pack_left, pack_right, GEMM; stats init + 2 stats passes

    def step_allgather(ev=None):
        k = k_state["k"] + 1
        with torch.cuda.stream(stream):
            if ev is not None:
                ev[0].record(stream)
            X = rdist.minplus_mul_allgather(A_rows, ag["ring"][k - 1], bounds)
            ag["ring"][k] = X
            prevs = [ag["ring"][k - a] for a in range(1, min(am, k - 1) + 1)]
            rd.rd_panel_stats(X, prevs, r0, am, stats, stream=stream)
            ag["ring"].pop(k - am - 1, None)
            if ev is not None:
                ev[1].record(stream)
            if world > 1:
                dist.all_reduce(stats, op=dist.ReduceOp.MIN)
            hstats.copy_(stats, non_blocking=True)
        stream.synchronize()
        k_state["k"] = k
        h = hstats.numpy()
        if k_state["found"] is None:
            dec = rd.rd_stats_decide(h, am, k)
            if dec:
                k_state["found"] = (k - dec[0], dec[0], dec[1])

    def step(ev=None):
        if args.form == "allgather":
            return step_allgather(ev)
        with torch.cuda.stream(stream):
            if ev is not None:
                ev[0].record(stream)
            if chain is not None:
                chain.step(stats)
            else:
                stats.copy_(neutral)
            if ev is not None:
                ev[1].record(stream)
            if world > 1:
                dist.all_reduce(stats, op=dist.ReduceOp.MIN)
            hstats.copy_(stats, non_blocking=True)
        stream.synchronize()
        k_state["k"] += 1
        h = hstats.numpy()
        if k_state["found"] is None:
            dec = rd.rd_stats_decide(h, am, k_state["k"])
            if dec:
                k_state["found"] = (k_state["k"] - dec[0], dec[0], dec[1])

    for _ in range(args.warmup):
        step()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    elapsed = t_start.elapsed_time(t_end) * 1e-3
    gemm_s = statistics.mean(a.elapsed_time(b) for a, b in evs) * 1e-3 if (chain is not None or args.form == "allgather") else 0.0
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    tmax = float(t.item())
    ops_total = float(N) ** 3 * args.steps
    value = ops_total / tmax / 1e9
    clocks = clk.summary()

    # roofline of the dominant kernel (the GEMM): algorithmic ops per launch / launch time
    ops_launch = float(r1 - r0) * N * N
    achieved = ops_launch / gemm_s / 1e9 if gemm_s > 0 else 0.0
    peak = SM_COUNT * PIPE_MINPLUS_PER_CLK_SM * SM_MAX_MHZ * 1e6 / 1e9
    dpx_peak = SM_COUNT * DPX_MINPLUS_PER_CLK_SM * SM_MAX_MHZ * 1e6 / 1e9
    mix_peak = SM_COUNT * probe["mixed_minplus_per_clk_sm"] * SM_MAX_MHZ * 1e6 / 1e9
    dpx_used = chain.gemm_variant if chain is not None and hasattr(chain, "gemm_variant") else None
    if chain is not None:
        chain.close()

    # e2e through the public API with host buffers (rd_power_sequence: host build, H2D, chain
    # to first detection, per-step stats D2H), wall clock, max over ranks
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        if world > 1:
            res = rdist.power_sequence(m, 50, am, broadcast=True)
        else:
            res = rd.rd_power_sequence(m, 50, am)
        torch.cuda.synchronize()
        te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        te = float(te.item())
        prods = res["k_stop"] - 1
        e2e = {"value": round(prods * float(N) ** 3 / te / 1e9, 3), "unit": "Gop/s",
               # the chain uploads A(G)'s CSC (colptr + entries), the device builds the operands
               "h2d_bytes_per_step": int(4 * (NNZ.get(m, 0) + N + 1)),
               "d2h_bytes_per_step": int(prods * rd.rd_stats_len(am) * 4),
               "step": "one rd_power_sequence(m, 50) call: build + upload A, chain to first detection",
               "seconds": round(te, 3), "k_stop": res["k_stop"],
               "triple": [res["n0"], res["alpha"], res["beta"]]}

    # dense power-step Gop/s at every order N = C_m (SURVEY §8(d) shapes and protocol: warm-up
    # steps through the chain's DPX tuning (A^4..A^11 at m = 8), then median and best of 10
    # individually event-timed steps A^(k-1) (x) A, k = 12..21)
    def timed(fn, warm=10, reps=10):
        with torch.cuda.stream(stream):
            for _ in range(warm):
                fn()
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for a, b in ev:
                a.record(stream)
                fn()
                b.record(stream)
        torch.cuda.synchronize()
        t = sorted(a.elapsed_time(b) * 1e-3 for a, b in ev)
        return statistics.median(t), t[0]

    gops_by_m = {}
    if rank == 0 and not args.no_e2e:
        for mm in args.gops_m:
            chm = rd.Chain(mm, alpha_max=am, stream=stream)
            nn = chm.N
            med, best = timed(chm.step)
            gops_by_m[str(mm)] = {"N": nn, "ms_per_step": round(med * 1e3, 4), "ms_best": round(best * 1e3, 4),
                                  "gops": round(float(nn) ** 3 / med / 1e9, 1),
                                  "gops_best": round(float(nn) ** 3 / best / 1e9, 1)}
            chm.close()

    # operand invariance: the dense kernel is data-oblivious, so the generic
    # product rd_minplus_mul (packing included) takes the same time on the real A^4 (x) A, on
    # A (x) A and on synthetic uniform [0, 1000] operands with 1% inf (seeds 0, 1, 2)
    invariance = None
    if rank == 0 and not args.no_e2e and args.invariance_m:
        from rd_inputs import operand
        mi = args.invariance_m
        chi = rd.Chain(mi, alpha_max=4, stream=stream)
        for _ in range(3):
            chi.step()
        A4 = torch.from_numpy(chi.read_rows(4)).to(dev)
        A1 = torch.from_numpy(chi.read_rows(1)).to(dev)
        chi.close()
        ni = A1.shape[0]
        C = torch.empty_like(A1)
        cases = {"A^4 (x) A": (A4, A1), "A (x) A": (A1, A1)}
        for sd in (0, 1, 2):
            cases[f"uniform[0,1000] 1% inf, seed {sd}"] = (
                torch.from_numpy(operand(ni, ni, sd)).to(dev), torch.from_numpy(operand(ni, ni, sd + 100)).to(dev))
        invariance = {"m": mi, "N": ni, "call": "rd_minplus_mul (pack + GEMM)", "ms_median": {}, "ms_best": {}}
        for name, (X, Y) in cases.items():
            med, best = timed(lambda: rd.rd_minplus_mul_ex(X, ni, Y, ni, C, ni, ni, ni, ni, stream=stream))
            invariance["ms_median"][name] = round(med * 1e3, 4)
            invariance["ms_best"][name] = round(best * 1e3, 4)
        v = list(invariance["ms_median"].values())
        invariance["spread"] = round(max(v) / min(v) - 1, 4)
        del cases, A4, A1, C
        # the 32-bit generic product (rd_minplus_mul32: entries beyond the int16 headroom) at the
        # same N, uniform [0, 2^29) with 1% inf
        X32 = torch.from_numpy(operand(ni, ni, 7, hi=2**29 - 1, inf=rd.RD_INF32, dtype=np.int32)).to(dev)
        Y32 = torch.from_numpy(operand(ni, ni, 8, hi=2**29 - 1, inf=rd.RD_INF32, dtype=np.int32)).to(dev)
        C32 = torch.empty_like(X32)
        med, best = timed(lambda: rd.rd_minplus_mul32(X32, Y32, C32, stream=stream))
        invariance["mul32"] = {"ms_median": round(med * 1e3, 4), "ms_best": round(best * 1e3, 4),
                               "gops": round(float(ni) ** 3 / med / 1e9, 1),
                               "data": "uniform [0, 2^29) int32, 1% inf, seeds 7, 8"}
        del X32, Y32, C32

    # the standalone reductions (a3 + a4 of the all-gather form, rd_panel_stats): diag-min and
    # the periodicity stats of a full m-sized power against alpha_max earlier ones, HBM-bound;
    # algorithmic bytes (1 + alpha_max) * 2 N^2 per call
    reductions = None
    if rank == 0 and not args.no_e2e:
        g = torch.Generator(device=dev).manual_seed(0)
        cur = torch.randint(100, 140, (N, N), dtype=torch.int16, device=dev, generator=g)
        prevs = [torch.randint(40 + 2 * a, 100, (N, N), dtype=torch.int16, device=dev, generator=g)
                 for a in range(am)]
        sr = torch.empty(rd.rd_stats_len(am), dtype=torch.int32, device=dev)
        med, best = timed(lambda: rd.rd_panel_stats(cur, prevs, 0, am, sr, stream=stream))
        byts = (1 + am) * 2 * float(N) * N
        hbm = _measured_hbm_gbs()
        reductions = {"call": "rd_panel_stats (diag min + periodicity stats of alpha = 1..alpha_max, one pass)",
                      "N": N, "alpha_max": am, "ms_median": round(med * 1e3, 4), "ms_best": round(best * 1e3, 4),
                      "algorithmic_bytes": int(byts), "achieved_gbs": round(byts / med / 1e9, 1),
                      "peak_gbs": hbm, "frac": round(byts / med / 1e9 / hbm, 4) if hbm else None,
                      "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy read+write)",
                      "data": "uniform int16 bands (seeded), fully finite"}
        del cur, prevs

    # time to periodicity per m (Alg 2 to first detection): build (words, A(G), upload,
    # packing) and chain (products + fused checks + per-step stats decision), max over ranks
    ttp = {}
    if not args.no_e2e:
        for mm in args.ttp_m:
            # one untimed run per small order and method first: the first launch of a kernel in
            # the process pays module loading (milliseconds against a 0.2 ms small-order chain)
            if world == 1 and mm <= 7:
                rd.rd_power_sequence(mm, 50, am)
                rd.rd_power_sequence(mm, 50, am, method=1)
            if world > 1:
                dist.barrier()
            # one GPU: the library's own loop (rd_power_sequence: speculative depth, C decisions);
            # several: the row-panel driver with the stats all_reduce
            res = (rd.rd_power_sequence(mm, 50, am) if world == 1
                   else rdist.power_sequence(mm, 50, am, broadcast=True))
            tt = torch.tensor([res["t_build"], res["t_chain"]], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            nn = rd.count_words(mm)
            ttp[str(mm)] = {"build_s": round(float(tt[0]), 6), "chain_s": round(float(tt[1]), 6),
                            "total_s": round(float(tt[0] + tt[1]), 6), "k_stop": res["k_stop"],
                            "triple": [res["n0"], res["alpha"], res["beta"]],
                            "chain_gops": round((res["k_stop"] - 1) * float(nn) ** 3 / float(tt[1]) / 1e9, 1)}
            # the structured step (NEXT-3: finite terms of the sparse right operand only),
            # same results; its Gop/s counts its own terms (rows x nnz(A) per step)
            if world > 1:
                dist.barrier()
            rs = (rd.rd_power_sequence(mm, 50, am, method=1) if world == 1
                  else rdist.power_sequence(mm, 50, am, method=1))
            ts = torch.tensor([rs["t_build"], rs["t_chain"]], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            assert (rs["n0"], rs["alpha"], rs["beta"]) == (res["n0"], res["alpha"], res["beta"])
            ttp[str(mm)]["structured"] = {"build_s": round(float(ts[0]), 6), "chain_s": round(float(ts[1]), 6),
                                          "total_s": round(float(ts[0] + ts[1]), 6),
                                          "terms_per_step": NNZ.get(mm, 0) * nn,
                                          "chain_gterms": round((rs["k_stop"] - 1) * NNZ.get(mm, 0) * nn
                                                                / float(ts[1]) / 1e9, 1)}

    # orders whose dense chain takes minutes: the structured chain only (NEXT-2/NEXT-3).
    # m = 11 (N = 191476, 73 GB per int16 power) from 4 ranks on: row panels of a ring of
    # alpha_max + 1 = 6 powers (the paper's alpha <= 5), 110 GB per rank at 4 GPUs
    structured_only = list(args.ttp_structured_only_m)
    if world >= 4 and 11 not in structured_only and not args.no_m11:
        structured_only.append(11)
    if not args.no_e2e:
        for mm in structured_only:
            if world > 1:
                dist.barrier()
            amm = min(am, 5) if mm >= 11 else am
            rs = (rd.rd_power_sequence(mm, 50, amm, method=1) if world == 1
                  else rdist.power_sequence(mm, 50, amm, method=1))
            ts = torch.tensor([rs["t_build"], rs["t_chain"]], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(ts, op=dist.ReduceOp.MAX)
            nn = rd.count_words(mm)
            ttp[str(mm)] = {"k_stop": rs["k_stop"], "triple": [rs["n0"], rs["alpha"], rs["beta"]], "alpha_max": amm,
                            "structured": {"build_s": round(float(ts[0]), 4), "chain_s": round(float(ts[1]), 4),
                                           "total_s": round(float(ts[0] + ts[1]), 4),
                                           "terms_per_step": NNZ.get(mm, 0) * nn,
                                           "chain_gterms": round((rs["k_stop"] - 1) * NNZ.get(mm, 0) * nn
                                                                 / float(ts[1]) / 1e9, 1)}}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = OracleSample(m)
        rows = smp.calibrate(args.cpu_seconds)
        rate, dt = smp.run(rows)
        cpu = {"value": round(rate, 3), "unit": "Gop/s", "cores": cores_used(), "kind": "oracle",
               "sample": f"{rows} sampled output rows of A^(k-1) (x) A(G), m={m}, dense i-j-k oracle, {dt:.1f} s"}
        # the oracle's own time to periodicity (Algorithm 2 with the INF-skipping product,
        # all host cores) beside the GPU's time_to_periodicity
        import oracle as O
        ttp_o = {}
        for mm in args.oracle_ttp_m:
            t0 = time.perf_counter()
            r = O.power_chain(mm, 50, am, 0)
            ttp_o[str(mm)] = {"seconds": round(time.perf_counter() - t0, 6), "triple": [r["n0"], r["alpha"], r["beta"]]}
        cpu["time_to_periodicity"] = ttp_o
        # SURVEY §8(d) oracle timings: the dense product at each small order (full N^3, same
        # OpenMP i-j-k loop) and the independent checkers on points of their domains
        dense = {}
        for mm in (3, 4, 5, 6, 7):
            Am = O.matrix(mm)
            BTm = np.ascontiguousarray(Am.T)
            t0 = time.perf_counter()
            O.minplus_bt(Am, BTm)
            dt = time.perf_counter() - t0
            dense[str(mm)] = {"N": Am.shape[0], "seconds": round(dt, 4),
                              "gops": round(float(Am.shape[0]) ** 3 / max(dt, 1e-9) / 1e9, 3)}
        cpu["dense_product_by_m"] = dense
        checks = {}
        for name, fn, a in (("X1 exhaustive f: V -> {0,1,2}", O.gamma_bruteforce3, (3, 5)),
                            ("X2 S2-subset brute force", O.gamma_s2subset, (4, 6)),
                            ("X3 row DP along the path", O.gamma_rowdp, (9, 8)),
                            ("X5 S2-pair trace DP", O.gamma_pairtrace, (4, 30))):
            t0 = time.perf_counter()
            v = fn(*a)
            checks[name] = {"m_n": list(a), "gamma": int(v), "seconds": round(time.perf_counter() - t0, 4)}
        cpu["checkers"] = checks
        cpu["host"] = {"cpu_model": _cpu_model(), "nproc": os.cpu_count()}

    if rank == 0:
        line = {
            "metric": "(min,+) Gop/s on A^(k-1) (x) A(G) at order N = C_m (power step with fused diag-min + periodicity test)",
            "value": round(value, 3), "unit": "Gop/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(tmax / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong",
            "vs_baseline": round(value / PAPER_K80_GOPS[m], 2) if m in PAPER_K80_GOPS else None,
            "dtype": "i16",
            "data": "deterministic A(G) of P_m (no dataset); powers computed in the timed steps",
            "config": {"workload": f"P_{m} box C_n: power step A^k = A^(k-1) (x) A(G), N = C_{m} = {N}",
                       "m": m, "N": N, "alpha_max": am, "parallelism": f"row panels x{world}", "form": args.form,
                       "backend": backend if world > 1 else None,
                       "l2": "operands (2N^2 B = %.0f MB each) exceed L2; no flush" % (2 * N * N / 1e6),
                       "k_range": [2 + args.warmup, 1 + args.warmup + args.steps]},
            "roofline": {"bound": "alu", "achieved": round(achieved, 1), "peak": round(peak, 1), "unit": "Gop/s",
                         "frac": round(achieved / peak, 4), "traffic": TRAFFIC.get(m) if args.form == "replicated" else None,
                         # compulsory DRAM bytes per launch: B (2N^2 B at int16), the panel's X and
                         # C, and the alpha_max earlier powers the fused periodicity test reads
                         "algorithmic_bytes": int(2 * N * N + (2 + am) * 2 * (r1 - r0) * N),
                         "kernel": "minplus_gemm_kernel<RP,STATS,3> (peer B)" if args.form == "peer"
                                   else "minplus_gemm_kernel<PM,STATS,%s%s>" % (
                                       dpx_used if dpx_used is not None else 3,
                                       ",TMA" if (N + 127) // 128 * 64 // 32 >= 64 else ""),
                         "peak_basis": "unit-count bound: 148 SMs x 192 (min,+)/clk/SM x 1965 MHz (alu 2 + fma 2 warp-instr/clk/SM, issue 4; "
                                       "best mix 1 VIADDMNMX.S16x2 : 1 [2 IMAD + 1 VIMNMX3.S16x2]; DESIGN.md 5)",
                         "dpx_issue_peak": round(dpx_peak, 1), "frac_of_dpx_issue_peak": round(achieved / dpx_peak, 4),
                         "dpx_issue_peak_basis": "DPX-only: 148 SMs x 128 (min,+)/clk/SM (VIADDMNMX.S16x2 at 2 warp-instr/clk/SM, measured) x 1965 MHz",
                         "mix_ceiling": round(mix_peak, 1), "frac_of_mix_ceiling": round(achieved / mix_peak, 4),
                         "mix_ceiling_basis": "register-tile probe of the GEMM's DPX+IMAD/VIMNMX3 mix (rd_alu_probe, live) x 148 SMs x 1965 MHz",
                         "probe": {k: round(v, 2) for k, v in probe.items()},
                         "dpx_cols": dpx_used},
            "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps * world,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "time_to_periodicity": ttp,
            "reductions": reductions,
            "gops_by_m": gops_by_m,
            "operand_invariance": invariance,
            "paper_context": {"k80_cumatrixtrop_gops_derived": PAPER_K80_GOPS.get(m),
                              "source": "BASELINE.md 1.1, 49 N^3 / Table 3 kernel time"},
        }
        if k_state["found"]:
            line["config"]["detected"] = list(k_state["found"])
        print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_command(argv, gpus: int, port: int):
    """The command that runs this script as `gpus` ranks of one node (one process per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def self_launch(args, argv) -> int | None:
    """`--gpus N > 1` without a launcher: re-run this script as N ranks under
    torch.distributed.run and return its exit status (None: nothing to launch).  Ranks must
    each have a GPU of their own unless the gloo test hook (RD_FORCE_DEVICE) is set."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl != "reference" and "RD_FORCE_DEVICE" not in os.environ:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible", file=sys.stderr)
            return 2
    import subprocess
    return subprocess.call(launch_command(argv, args.gpus, _free_port()))


def main():
    args = parse()
    rc = self_launch(args, sys.argv[1:])
    if rc is not None:
        sys.exit(rc)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started {world} rank(s)", file=sys.stderr)
        sys.exit(2)
    # test hooks: several ranks on one GPU with host-side (gloo) collectives; never used for
    # a reported number (the line then says so in config.backend)
    if "RD_FORCE_DEVICE" in os.environ:
        local_rank = int(os.environ["RD_FORCE_DEVICE"])
    backend = os.environ.get("RD_DIST_BACKEND", "nccl")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank, backend)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
