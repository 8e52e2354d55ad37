#!/usr/bin/env python
"""Benchmark: full Pauli decomposition of a dense 2^N x 2^N complex128 matrix on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--qubits 14]

A step is one full decomposition (all 4^N coefficients) of the N=14 matrix of BASELINE.json
configs[4] (the reference's seeded uniform[-1,1) generator, 4 GiB), on the Gray-code path:
K1 diagonal gather + K2 Gray-code FP64 sums (+ NCCL broadcast of G and gather of the
coefficient runs when N > 1, one process per GPU under torchrun). Rank 0 prints one JSON line.

--impl reference times the reference's own CPU implementation (oracle/_ref/libpdref.so: the
reference's proj/src compiled unmodified, coeff_fast over all host threads) on a seeded
sample of X-masks of the same workload, scaled per coefficient.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ACCEPT_SEED = 20260823  # proj/tests/acceptance.cpp:30
METRIC = "pauli_coeffs_per_sec"
UNIT = "coeff/s"
SM_COUNT = 148
FP64_LANES_PER_SM = 64


def parse_args():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--qubits", type=int, default=14)
    ap.add_argument("--path", choices=["gray", "wht"], default="gray")
    ap.add_argument("--mode", choices=["nccl", "nccl-serial", "peer"], default="nccl",
                    help="N>1 data path: NCCL pipeline (diagonal chunks scattered in walk order, "
                         "sub-blocks gathered while the next computes), serial NCCL broadcast + "
                         "gather, or CUDA-IPC peer memory (K1 reads rank 0's G, K2 stores into "
                         "rank 0's output)")
    ap.add_argument("--sample-masks", type=int, default=64,
                    help="X-masks in the CPU sample (>= 8); 64 = 1,048,576 coefficients, ~10 s on 16 threads")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the N=12 and WHT side lines")
    return ap.parse_args()


def workload_config(nq: int, world: int, path: str, mode: str = "nccl") -> dict:
    return {
        "workload": f"full decomposition N={nq} (BASELINE configs[4])" if nq == 14
        else f"full decomposition N={nq}",
        "num_qubits": nq,
        "coefficients": 4**nq,
        "matrix": f"random_matrix({nq}, matrix_seed({ACCEPT_SEED},{nq},0)): uniform[-1,1) complex128, "
                  f"{16 * 4**nq / 2**30:g} GiB (reference generator, bit-exact on device)",
        "path": "gray-code K1+K2" if path == "gray" else "walsh-hadamard K1+K4",
        "parallelism": f"xmask-shard x{world}" + ({
            "nccl": " (NCCL pipeline: rank 0 gathers each rank's diagonals one walk chunk at a time and "
                    "sends them in walk order, walk segments chase the chunks, finished sub-blocks "
                    "are sent to rank 0 while the next computes)",
            "nccl-serial": " (NCCL broadcast G + grouped send/recv gather)",
            "peer": " (CUDA-IPC peer memory: K1 reads rank 0's G, K2 stores into rank 0's output)",
        }[mode] if world > 1 else ""),
        "l2": "inputs (4 GiB G, 4 GiB diagonals) exceed the 126 MB L2; no flush needed" if nq >= 12
        else "inputs smaller than L2",
    }


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, local_rank: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        self.index = vis.split(",")[local_rank] if vis else str(local_rank)
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", self.index], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, ValueError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "power_w_max": max(power) if power else None,
                "samples": len(sm),
                "reasons": sorted(reasons)}


# ---------------------------------------------------------------- reference arm

def cpu_sample_masks(nq: int, k: int) -> list:
    import numpy as np
    rng = np.random.default_rng(ACCEPT_SEED + nq)
    return sorted(int(x) for x in rng.choice(2**nq, size=min(k, 2**nq), replace=False))


class CpuBaseline:
    """The reference's CPU path on this host: coeff_fast on every string of k seeded X-masks
    (ascending n, contiguous split over all hardware threads), BASELINE.md §2."""

    def __init__(self, nq: int, k: int, host_matrix=None):
        import numpy as np
        from oracle import oracle as O
        self.nq = nq
        self.ref = O.reference()
        self.kind = "reference" if self.ref is not None else "port"
        self.masks = cpu_sample_masks(nq, k)
        self.ns = O.xmask_sample_indices(nq, self.masks)
        seed = O.port().matrix_seed(ACCEPT_SEED, nq, 0)
        if self.ref is not None:
            self.cores = self.ref.cores
            self.h = self.ref.matrix(host_matrix) if host_matrix is not None else \
                self.ref.random_matrix_handle(nq, seed)
        else:
            self.cores = os.cpu_count() or 1
            self.port = O.port()
            self.g = host_matrix if host_matrix is not None else self.port.random_matrix(nq, seed)
        self.sample = (f"{len(self.masks)} seeded X-masks x all {2**nq} Z-masks = {self.ns.size} "
                       f"coefficients of the N={nq} workload via "
                       + ("reference coeff_fast (proj/src, -O3)" if self.kind == "reference"
                          else "oracle port of coeff_fast")
                       + f" on {self.cores} threads; throughput scales linearly to all 4^N")

    def run_once(self) -> float:
        t0 = time.perf_counter()
        if self.kind == "reference":
            self.out = self.ref.coeff_batch(self.h, self.ns, threads=self.cores)
        else:
            self.out = self.port.coeff_batch(self.g, self.ns, threads=self.cores)
        return time.perf_counter() - t0


def n12_cpu_baseline(g, gpu_out):
    """BASELINE configs[3] on the host: the reference's own decompose_parallel
    (proj/src/decompose.cpp:95-131, 205-211) over all 4^12 coefficients on every hardware
    thread, once, timed with a wall clock like bench.cpp:105-108; its output must equal the
    GPU's bit for bit."""
    import numpy as np
    from oracle import oracle as O
    ref = O.reference()
    if ref is None:
        return {"unavailable": "oracle/_ref not built"}
    h = ref.matrix(g)
    t0 = time.perf_counter()
    c = ref.decompose(h, threads=ref.cores)
    sec = time.perf_counter() - t0
    return {"value": c.size / sec, "unit": UNIT, "cores": ref.cores, "kind": "reference",
            "sample": "full N=12 decomposition (16,777,216 coefficients) via reference "
                      "decompose_parallel (proj/src, -O3), one run", "seconds": sec,
            "matches_gpu_full_array": bool(np.array_equal(c, gpu_out))}


def small_cpu_baseline(g, gpu_out, ns=None, reps=3):
    """BASELINE configs[0-2] on the host, the reference's own code on every hardware thread:
    decompose_parallel (full decompositions) or coeff_fast over a string batch (contiguous split),
    best of `reps` wall-clock runs; its output must equal the GPU's bit for bit."""
    import numpy as np
    from oracle import oracle as O
    ref = O.reference()
    if ref is None:
        return {"unavailable": "oracle/_ref not built"}
    h = ref.matrix(g)
    best, c = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        c = ref.decompose(h, threads=ref.cores) if ns is None else ref.coeff_batch(h, ns, threads=ref.cores)
        sec = time.perf_counter() - t0
        best = sec if best is None else min(best, sec)
    return {"value": c.size / best, "unit": UNIT if ns is None else "strings/s", "cores": ref.cores,
            "kind": "reference", "seconds": best,
            "sample": ("full decomposition via reference decompose_parallel" if ns is None
                       else f"{ns.size} strings via reference coeff_fast") + " (proj/src, -O3), best of "
                      + str(reps),
            "matches_gpu": bool(np.array_equal(c, gpu_out))}


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # only rank 0 times the CPU reference; other ranks exit without work
    nq = args.qubits
    base = CpuBaseline(nq, max(8, args.sample_masks))
    for _ in range(args.warmup):
        base.run_once()
    times = [base.run_once() for _ in range(args.steps)]
    per_step = sum(times) / len(times)
    value = base.ns.size / per_step
    line = {
        "impl": "reference",
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step * 1e3,
        "ms_per_full_decomposition_est": 4**nq / value * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(nq, args.gpus, "gray"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": base.cores, "kind": base.kind,
                         "sample": base.sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm

def sd_ptr(buf) -> int:
    return buf.data_ptr() if hasattr(buf, "data_ptr") else int(buf)


def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2401_16378_b200 as pd
    from paper_2401_16378_b200.sharding import ShardPlan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    nq = args.qubits
    dim = 1 << nq
    plan = ShardPlan(nq, world, rank)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    pd.set_device(local_rank)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    G = torch.empty((dim, dim), dtype=torch.complex128, device=dev)
    pd_seed = pd.matrix_seed(ACCEPT_SEED, nq, 0)  # the reference generator's seed (bench.cpp:42-46)
    if rank == 0:
        pd.device.random_matrix(nq, pd_seed, G.data_ptr(), sptr)
    from paper_2401_16378_b200.sharding import ShardedDecomposer, scratch_tensor
    out = torch.empty(4**nq, dtype=torch.complex128, device=dev) if rank == 0 else None
    if world == 1:
        # one GPU: K1 and K2 launched here so that they can be timed apart
        diag = scratch_tensor(nq, plan.x_count, args.path, dev)
        sd = None
    else:
        # the sharding layer: NCCL pipeline (diagonal chunks scattered in walk order, walk
        # segments chasing them, finished sub-blocks gathered while the next computes), the
        # serial NCCL mode, or CUDA-IPC peer memory
        diag = None
        sd = ShardedDecomposer(nq, dev, mode=args.mode, path=args.path)
        if sd.mode == "peer":   # rank 0's G and output mapped once, outside the timed region
            sd.peer_buffers(G, out)
            torch.cuda.synchronize()
            barrier()

    def step(path, ev=None):
        if ev is not None:
            ev[0].record(stream)
        if world > 1:  # the whole sharded step (its kernels and transfers on the layer's streams)
            if ev is not None:
                ev[1].record(stream)
            sd(G, out)
            if ev is not None:
                ev[2].record(stream)
            return
        gp, dp = G.data_ptr(), out.data_ptr()
        if path == "gray":  # K1 and K2 timed separately
            pd.device.diag_gather(nq, gp, plan.x0, plan.x_count, diag.data_ptr(), sptr)
            if ev is not None:
                ev[1].record(stream)
            pd.device.xmask_coeffs(nq, diag.data_ptr(), plan.x0, plan.x_count, plan.run_bits,
                                   dp, "global", path, sptr)
        else:  # fused two-pass WHT straight from G
            if ev is not None:
                ev[1].record(stream)
            pd.device.shard_coeffs(nq, gp, plan.x0, plan.x_count, plan.run_bits,
                                   dp, "global", diag.data_ptr(), path, sptr)
        if ev is not None:
            ev[2].record(stream)

    def timed(path, steps, warmup, sample_clocks=False):
        for _ in range(warmup):
            step(path)
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(local_rank) if sample_clocks else None
        if clocks:
            clocks.start()
        barrier()
        torch.cuda.synchronize()
        l0 = pd.launch_count()
        t0.record(stream)
        for s in range(steps):
            step(path, evs[s])
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        launches = pd.launch_count() - l0
        ck = clocks.stop() if clocks else None
        ms = max_over_ranks(t0.elapsed_time(t1))
        k1 = sum(e[0].elapsed_time(e[1]) for e in evs) / steps
        k2 = sum(e[1].elapsed_time(e[2]) for e in evs) / steps
        return ms, k1, k2, launches, ck

    # FP64-add probe (peak context) and the headline measurement
    probe = pd.fp64_add_probe(local_rank)
    ms, k1_ms, k2_ms, launches, clocks = timed(args.path, args.steps, args.warmup, sample_clocks=True)
    per_step_ms = ms / args.steps
    value = 4**nq / (per_step_ms / 1e3)

    # roofline of the dominant kernel (K2 Gray: FP64-add bound; K4 WHT: HBM bound)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        pass
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(f"N{nq}_{args.path}_x{world}")
    except (OSError, ValueError):
        pass
    if args.path == "gray":
        dadd = k2_dadd(nq) / world
        ref_dadd = 2.0 * dim * (4**nq / world)  # the reference's walk: 2 adds x 2^N terms each
        achieved = dadd / (k2_ms / 1e3) / 1e12
        peak = SM_COUNT * FP64_LANES_PER_SM * sm_max * 1e6 / 1e12
        roofline = {"bound": "fp64", "kernel": "gray_share_c_kernel (K2s-c)" if nq >= 13 else "gray_share_kernel (K2s)",
                    "achieved": achieved,
                    "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                    "algorithmic": f"DADDs the Gray kernel executes: the reference's 2*2^N per coefficient less the "
                                   f"shared walk prefixes (x 171/256) = {dadd:.4g} per launch",
                    "reference_walk_equiv_tflops": ref_dadd / (k2_ms / 1e3) / 1e12,
                    "peak_source": f"nominal FP64 add: {SM_COUNT} SM x {FP64_LANES_PER_SM} lanes x "
                                   f"{sm_max:g} MHz (MEASURED_PEAKS.json has no FP64 entry)",
                    "probe_tflops": probe / 1e12, "frac_of_probe": achieved / (probe / 1e12),
                    "k1_gather_ms": k1_ms, "k2_ms": k2_ms,
                    "k1_gather_gbs": 32.0 * 4**nq / world / (k1_ms / 1e3) / 1e9 if k1_ms > 0 else None}
        if world > 1:
            roofline["timed"] = ("the whole sharded step on each rank (its K1/K2 segments and the NCCL "
                                 "transfers they overlap), max over ranks: a lower bound on the kernel's rate")
            roofline["k2_ms"] = k2_ms = ms / args.steps
            roofline.pop("k1_gather_ms")
            roofline.pop("k1_gather_gbs")
            roofline["achieved"] = achieved = dadd / (k2_ms / 1e3) / 1e12
            roofline["frac"] = achieved / peak
            roofline["frac_of_probe"] = achieved / (probe / 1e12)
            roofline["reference_walk_equiv_tflops"] = ref_dadd / (k2_ms / 1e3) / 1e12
    else:
        byts = 32.0 * 4**nq / world
        achieved = byts / ((k1_ms + k2_ms) / 1e3) / 1e9
        peak = float(peaks.get("hbm_gbs", 6542.7))
        roofline = {"bound": "hbm", "kernel": "K4 fused WHT (wht_gather_lo + wht_hi_out)", "achieved": achieved,
                    "peak": peak, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": per_step_ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_config(nq, world, args.path, sd.mode if sd is not None else args.mode),
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clocks,
    }

    # ---- cpu_baseline: the reference on this host, rank 0 at N=1 only
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        gh = G.cpu().numpy()
        base = CpuBaseline(nq, max(8, args.sample_masks), host_matrix=gh)
        secs = base.run_once()
        # the device result must match the reference on the sampled strings, value for value
        got = out[torch.from_numpy(base.ns.astype(np.int64)).to(dev)].cpu().numpy() \
            if args.path == "gray" else None
        line["cpu_baseline"] = {"value": base.ns.size / secs, "unit": UNIT, "cores": base.cores,
                                "kind": base.kind, "sample": base.sample,
                                "seconds": secs}
        if got is not None:
            line["cpu_baseline"]["sample_matches_gpu"] = bool(np.all(got == base.out))
        del gh, base

    # ---- side measurements: N=12 (the metric's other size) and the WHT path
    if not args.no_extras:
        if args.path == "gray":
            ms_w, k1w, k4w, _, _ = timed("wht", args.steps, max(3, args.warmup))
            byts = 32.0 * 4**nq / world
            line["wht_path"] = {"value": 4**nq / (ms_w / args.steps / 1e3), "unit": UNIT,
                                "ms_per_step": ms_w / args.steps,
                                "roofline": {"bound": "hbm", "achieved": byts / ((k1w + k4w) / 1e3) / 1e9,
                                             "peak": float(peaks.get("hbm_gbs", 6542.7)), "unit": "GB/s",
                                             "algorithmic": "32*4^N B (read G once, write coefficients once)",
                                             "kernel": "K4 fused two-pass WHT", "k4_ms": k4w}}
            line["wht_path"]["roofline"]["frac"] = (line["wht_path"]["roofline"]["achieved"]
                                                    / line["wht_path"]["roofline"]["peak"])
            # recompose (the inverse) of the last step's coefficients into a second
            # matrix, checked against G: the chunked inverse WHT passes, HBM-bound at 32*4^N B
            if world == 1 and args.path == "gray":
                scr = diag if diag is not None else scratch_tensor(nq, plan.x_count, "wht", dev)
                g2 = torch.empty_like(G)

                def rec():
                    pd.device.recompose(nq, out.data_ptr(), g2.data_ptr(), scr.data_ptr(), sptr)
                for _ in range(3):
                    rec()
                torch.cuda.synchronize()
                ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                ea.record(stream)
                for _ in range(args.steps):
                    rec()
                eb.record(stream)
                torch.cuda.synchronize()
                rms = ea.elapsed_time(eb) / args.steps
                err = float(torch.max(torch.abs(g2 - G)))
                del g2
                hbm = float(peaks.get("hbm_gbs", 6542.7))
                line["recompose"] = {"ms_per_step": rms, "unit": "GB/s",
                                     "roofline": {"bound": "hbm", "achieved": 32.0 * 4**nq / (rms / 1e3) / 1e9,
                                                  "peak": hbm, "unit": "GB/s",
                                                  "frac": 32.0 * 4**nq / (rms / 1e3) / 1e9 / hbm,
                                                  "algorithmic": "32*4^N B (read coefficients, write G)"},
                                     "max_abs_err_vs_G": err}
        if world == 1 and rank == 0:
            line["side_configs"] = side_configs(pd, dev, stream, sptr, peaks, not args.no_cpu_baseline)

    # ---- e2e through the public API with pinned host buffers (H2D + D2H inside)
    if not args.no_e2e:
        del diag
        e2e = run_e2e(args, pd, plan, G, out, dev, stream, barrier, max_over_ranks, world, rank, sd)
        wht_e2e = e2e.pop("wht_path_e2e", None)
        line["e2e"] = e2e
        if wht_e2e is not None and "wht_path" in line:
            line["wht_path"]["e2e"] = wht_e2e

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def k2_dadd(nq):
    """FP64 adds one full Gray-path decomposition executes. K2s (pd_k2share.cu, N >= 9) walks
    16 Z-masks per thread that share walk prefixes: over the 16 regions of 2^(N-4) steps the live
    chains are 1, 2, 4, 4, 8 x 4, 16 x 8 (171 of 256), two adds (re, im) per chain and step, for
    2^(N-4) threads per X-mask and 2^N X-masks. Below N=9 K2 walks every chain: 2 * 8^N."""
    if nq >= 9:
        return 2.0 * 171 * 2.0 ** (3 * nq - 8)
    return 2.0 * 8.0**nq


def host_e2e(pd, g, steps, path="gray"):
    """pd.decompose on host buffers, wall clock per call after one warm-up: pinned in and out
    (`e2e`, the bench contract's form), and the reference binding's normal call on a plain numpy
    array returning a new array (`pageable`, bindings/module.cpp:21-42)."""
    import numpy as np
    import torch
    nq = g.shape[0].bit_length() - 1
    gp_t = torch.empty(g.shape, dtype=torch.complex128, pin_memory=True)
    op_t = torch.empty(4**nq, dtype=torch.complex128, pin_memory=True)
    gp, op = gp_t.numpy(), op_t.numpy()
    gp[...] = g
    gpage = np.array(g, copy=True)

    def clock(fn):
        fn()
        t = []
        for _ in range(steps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        return sum(t) / len(t)

    pinned = clock(lambda: pd.decompose(gp, out=op, path=path))
    page_new = clock(lambda: pd.decompose(gpage, path=path))
    nbytes = 16 * 4**nq
    return {"value": 4**nq / pinned, "unit": UNIT, "ms_per_step": pinned * 1e3,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "api": "decompose(pinned numpy, out=pinned numpy)",
            "pageable": {"value": 4**nq / page_new, "unit": UNIT, "ms_per_step": page_new * 1e3,
                         "api": "decompose(numpy array) -> new numpy array (pageable in and out)"}}


def side_configs(pd, dev, stream, sptr, peaks, cpu_n12=True):
    """The other BASELINE configs on one GPU, device-resident, CUDA events, 3 warm-ups:
    configs[3] (full N=12 decomposition, the metric's other size), configs[1] (65,536 batched
    single strings at N=10), configs[2] (full N=10 Hermitian) and configs[0] (full N=6)."""
    import numpy as np
    import torch

    def ev_time(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    res = {}
    nq = 12
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=dev)
    gen = np.random.default_rng(12)
    g.copy_(torch.from_numpy(gen.standard_normal((2**nq, 2**nq)) + 1j * gen.standard_normal((2**nq, 2**nq))))
    out = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    scr = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    ms = ev_time(lambda: pd.device.decompose(nq, g.data_ptr(), out.data_ptr(), scr.data_ptr(), "gray", sptr), 10)
    dadd = k2_dadd(nq)
    peak = SM_COUNT * FP64_LANES_PER_SM * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    res["n12_full_gray"] = {"config": "BASELINE configs[3]: full N=12, N(0,1) complex128",
                            "value": 4**nq / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                            "fp64_frac_incl_k1": dadd / (ms / 1e3) / peak}
    # the same matrix through the public API from host memory, pinned and pageable
    res["n12_full_gray"]["e2e"] = host_e2e(pd, g.cpu().numpy(), 10)
    if cpu_n12:
        res["n12_full_gray"]["cpu_baseline"] = n12_cpu_baseline(g.cpu().numpy(), out.cpu().numpy())
    nq = 10
    g = torch.empty((2**nq, 2**nq), dtype=torch.complex128, device=dev)
    g.copy_(torch.from_numpy(gen.standard_normal((2**nq, 2**nq)) + 1j * gen.standard_normal((2**nq, 2**nq))))
    ns = torch.from_numpy(gen.integers(0, 4**nq, 65536).astype(np.int64)).to(dev)
    o = torch.empty(65536, dtype=torch.complex128, device=dev)
    ms = ev_time(lambda: pd.device.coeff_batch(nq, g.data_ptr(), ns.data_ptr(), 65536, False, o.data_ptr(), sptr), 20)
    res["n10_strings"] = {"config": "BASELINE configs[1]: 65,536 random strings of an N=10 matrix",
                          "value": 65536 / (ms / 1e3), "unit": "strings/s", "ms_per_step": ms,
                          "kernel": "K3b: bucketed by X-mask, one CTA per bucket over its staged diagonal"}
    if cpu_n12:
        res["n10_strings"]["cpu_baseline"] = small_cpu_baseline(
            g.cpu().numpy(), o.cpu().numpy(), ns=ns.cpu().numpy().astype(np.uint64))
    # configs[2]: full N=10 decomposition of a Hermitian matrix (imaginary parts ~0)
    a = gen.standard_normal((2**nq, 2**nq)) + 1j * gen.standard_normal((2**nq, 2**nq))
    h = torch.from_numpy((a + a.conj().T) / 2).to(dev)
    out = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    scr = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    ms = ev_time(lambda: pd.device.decompose(nq, h.data_ptr(), out.data_ptr(), scr.data_ptr(), "gray", sptr), 20)
    res["n10_hermitian_full"] = {"config": "BASELINE configs[2]: full N=10 decomposition of (A+A^H)/2",
                                 "value": 4**nq / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
                                 "max_abs_imag": float(torch.max(torch.abs(out.imag)))}
    if cpu_n12:
        res["n10_hermitian_full"]["cpu_baseline"] = small_cpu_baseline(h.cpu().numpy(), out.cpu().numpy())
    # configs[0]: full N=6 decomposition (latency of one small call on the device)
    nq = 6
    g6 = torch.from_numpy(gen.standard_normal((64, 64)) + 1j * gen.standard_normal((64, 64))).to(dev)
    o6 = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    s6 = torch.empty(4**nq, dtype=torch.complex128, device=dev)
    ms = ev_time(lambda: pd.device.decompose(nq, g6.data_ptr(), o6.data_ptr(), s6.data_ptr(), "gray", sptr), 50)
    res["n6_full"] = {"config": "BASELINE configs[0]: full N=6 decomposition", "value": 4**nq / (ms / 1e3),
                      "unit": UNIT, "ms_per_step": ms}
    if cpu_n12:
        res["n6_full"]["cpu_baseline"] = small_cpu_baseline(g6.cpu().numpy(), o6.cpu().numpy(), reps=20)
    return res


def run_e2e(args, pd, plan, G, out, dev, stream, barrier, max_over_ranks, world, rank, sd=None):
    """The user-facing call on host memory. N=1: paper_2401_16378_b200.decompose(G_host, out=...)
    (C ABI pd_decompose: H2D, K1, K2, D2H). N>1: rank 0 uploads G, ShardedDecomposer runs the
    broadcast/compute/gather, rank 0 downloads the coefficients."""
    import torch

    import numpy as np
    nq = args.qubits
    nbytes = 16 * 4**nq
    steps = max(1, min(args.steps, 5))
    if world == 1:
        def clock(fn):
            fn()  # warm-up: the context allocates its buffers (and staging slots)
            t = []
            for _ in range(steps):
                t0 = time.perf_counter()
                r = fn()
                t.append(time.perf_counter() - t0)
                del r
            return sum(t) / len(t)

        def entry(per, api):
            return {"value": 4**nq / per, "unit": UNIT, "ms_per_step": per * 1e3,
                    "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes, "api": api}

        wht = args.path == "gray" and not args.no_extras
        gh_t = torch.empty(G.shape, dtype=torch.complex128, pin_memory=True)
        gh_t.copy_(G)
        oh_t = torch.empty(4**nq, dtype=torch.complex128, pin_memory=True)
        gh, oh = gh_t.numpy(), oh_t.numpy()
        res = entry(clock(lambda: pd.decompose(gh, out=oh, path=args.path)),
                    "paper_2401_16378_b200.decompose(pinned numpy, out=pinned numpy)")
        if wht:
            # the separately reported WHT path through the same call (per-block tile uploads
            # overlapping the downloads)
            res["wht_path_e2e"] = entry(clock(lambda: pd.decompose(gh, out=oh, path="wht")),
                                        "decompose(pinned numpy, out=pinned numpy, path='wht')")
        # the reference binding's normal call: a plain (pageable) numpy matrix in, a new numpy
        # array out (bindings/module.cpp:21-42), served through the pinned slot rings of
        # csrc/pd_stage.cu
        gpage = np.array(gh, copy=True)
        del gh, oh, gh_t, oh_t
        res["pageable"] = entry(clock(lambda: pd.decompose(gpage, path=args.path)),
                                "paper_2401_16378_b200.decompose(numpy array) -> new numpy array")
        if wht:
            res["wht_path_e2e"]["pageable"] = entry(
                clock(lambda: pd.decompose(gpage, path="wht")),
                "decompose(numpy array, path='wht') -> new numpy array")
        return res
    from paper_2401_16378_b200.sharding import ShardedDecomposer
    if sd is None:
        sd = ShardedDecomposer(nq, dev, path=args.path, mode=args.mode)
    gh_t = oh_t = None
    if rank == 0:
        gh_t = torch.empty(G.shape, dtype=torch.complex128, pin_memory=True)
        gh_t.copy_(G)
        oh_t = torch.empty(4**nq, dtype=torch.complex128, pin_memory=True)

    def one():
        if rank == 0:
            G.copy_(gh_t, non_blocking=True)
        sd(G, out)
        if rank == 0:
            oh_t.copy_(out, non_blocking=True)
        torch.cuda.synchronize()

    one()
    barrier()
    times = []
    for _ in range(steps):
        barrier()
        t0 = time.perf_counter()
        one()
        barrier()
        times.append(time.perf_counter() - t0)
    per = max_over_ranks(sum(times) / len(times))
    return {"value": 4**nq / per, "unit": UNIT,
            "h2d_bytes_per_step": nbytes if rank == 0 else 0,
            "d2h_bytes_per_step": nbytes if rank == 0 else 0, "ms_per_step": per * 1e3,
            "api": "paper_2401_16378_b200.sharding.ShardedDecomposer with pinned host G/out on rank 0"}


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: start the N ranks (one process per
    GPU) under torch.distributed.run on this node, 127.0.0.1 rendezvous, same arguments."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args))
    if args.gpus > 1:
        # NCCL's communicator setup on stderr (stdout keeps rank 0's one JSON line): rank and
        # nranks of every communicator, for the driver's check
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    run_ours(args)


if __name__ == "__main__":
    main()
