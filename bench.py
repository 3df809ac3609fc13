"""bench.py -- FIF hot-path throughput on B200 (BASELINE.json metric: signal samples decomposed/sec,
fp64 FIF, all IMFs; % of HBM roofline).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg1]

A "step" is one fif_decompose of the whole batch (every step of the hot path: forward rfft, extrema,
filter length, window spectrum, stopping search, damping + IFFT + remainder update, outer loop, for all
IMFs of all signals).  N=1 workload: config 1 (4096 signals x n=4096, fp64).  N>1 (torchrun): each rank
decomposes its own 4096 signals (weak scaling, no data-path collective: signals are independent).

Timing: W untimed warm-up steps, then K steps bracketed by barrier + cuda synchronize, CUDA events on the
launching stream, max over ranks.  Inputs (128 MiB) + outputs (1.4 GiB) per step exceed the 126 MB L2.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "signal samples decomposed/sec (fp64 FIF, all IMFs)"
UNIT = "samples/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback (only if MEASURED_PEAKS.json is absent)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--emulate", type=int, default=0,
                    help="cfg3 on one GPU: run the distributed algorithm with this many emulated ranks")
    ap.add_argument("--n", type=int, default=1 << 14, help="signal length for cfg4 (fp32 sweep)")
    ap.add_argument("--batch", type=int, default=None, help="signals per rank (default: the config's)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="default run: skip the config-2 line")
    ap.add_argument("--no-eig", action="store_true",
                    help="resident plans: evaluate the window spectrum per IMF instead of the per-L table")
    return ap.parse_args()


def workload(cfg, batch, n4=1 << 14):
    """(n, batch per rank, delta, dtype) of a BASELINE.json config."""
    from paper_1802_01359_b200 import signals

    if cfg == "cfg4":
        return n4, signals.cfg4_batch(n4) if batch is None else batch, 1e-3, "f32"
    if cfg == "cfg3":
        return (signals.CONFIGS["cfg3"]["n"] if n4 is None or n4 == 1 << 14 else n4), 1, 1e-3, "f64"
    c = signals.CONFIGS[cfg]
    B = c["batch"] if batch is None else batch
    return c["n"], B, c["delta"], c["dtype"]


def hbm_peak():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg, n, delta, budget_s=12.0, max_signals=256, n4=None):
    """The oracle as it stands (TD literal iteration, OpenMP over signals) on a bounded sample of the
    same workload: the first S signals of the batch, S grown until >= budget_s of CPU work."""
    import oracle
    from paper_1802_01359_b200 import signals

    ncores = oracle.num_threads()
    if cfg == "cfg3":  # one 2^26 signal: the literal iteration is out of reach; the paper's direct form
        from oracle import direct_form as df  # (numpy FFT, linear N scan) on a 2^22 cfg3-recipe signal

        m = 1 << 22
        s = signals.cfg3_signal(0, n=m)
        t0 = time.perf_counter()
        df.decompose(s, delta=delta)
        t_total = time.perf_counter() - t0
        return {"value": m / t_total, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"one cfg3-recipe signal of n=2^22 through oracle/direct_form.py (numpy FFT direct form, "
                          f"linear N scan), {t_total:.1f} s, single-threaded numpy"}
    if cfg == "cfg2":  # the literal iteration costs ~3e11 FMAs per 65536-sample signal: the direct form
        from oracle import direct_form as df

        done, t_total = 0, 0.0
        while t_total < budget_s and done < max_signals:
            s = signals.make_batch("cfg2", batch=1, start=done)[0]
            t0 = time.perf_counter()
            df.decompose(s, delta=delta)
            t_total += time.perf_counter() - t0
            done += 1
        return {"value": done * n / t_total, "unit": UNIT, "cores": 1, "kind": "oracle",
                "sample": f"first {done} signals of cfg2 (n={n}) through oracle/direct_form.py (numpy FFT direct "
                          f"form, linear N scan), {t_total:.1f} s, single-threaded numpy"}
    done, t_total, start = 0, 0.0, 0
    chunk = max(ncores, 8)
    while t_total < budget_s and done < max_signals:
        s = signals.make_batch(cfg, batch=chunk, start=start, n=n4).astype(np.float64)
        t0 = time.perf_counter()
        oracle.decompose(s, delta=delta)
        t_total += time.perf_counter() - t0
        done += chunk
        start += chunk
    return {"value": done * n / t_total, "unit": UNIT, "cores": ncores, "kind": "oracle",
            "sample": f"first {done} signals of {cfg} (n={n}), time-domain oracle (literal iteration), "
                      f"{t_total:.1f} s on {ncores} host threads"}


def rank_start(rank: int, per_rank: int) -> int:
    """Weak scaling: rank r decomposes signals [r*B, (r+1)*B) of the generator stream (no data-path collective)."""
    return rank * per_rank


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Max of a per-rank time over all ranks (the step time of the whole job)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def share_uid(rank: int, make_uid) -> bytes:
    """Rank 0 makes the NCCL unique id (fif_nccl_unique_id); every rank receives it (torch.distributed)."""
    import torch.distributed as tdist

    obj = [make_uid() if rank == 0 else None]
    tdist.broadcast_object_list(obj, src=0)
    return obj[0]


def time_block(full, rank: int, world: int):
    """Config 3 sharding: rank r owns samples [r n/world, (r+1) n/world) of the one long signal."""
    return np.ascontiguousarray(full.reshape(world, -1)[rank])


def self_launch(args) -> int:
    """`--gpus N` (N > 1) without torchrun: re-run this command under torch.distributed.run with N local ranks
    (127.0.0.1 rendezvous, a free port) and return its exit code; rank 0 prints the JSON line as usual."""
    import socket

    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    print(f"[bench] --gpus {args.gpus} without torchrun: launching {args.gpus} ranks", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        if args.gpus != world:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        if args.impl == "ours":  # NCCL's init lines (ranks, NVLink/NVLS topology) on stderr for the record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        backend = "nccl" if args.impl == "ours" else "gloo"
        dist.init_process_group(backend=backend)
    print(f"[bench] rank {rank}/{world} (local {local}) impl={args.impl}", file=sys.stderr, flush=True)
    return world, rank, local


def run_reference(args, world, rank):
    """--impl reference: the oracle (TD literal iteration) on the host cores, bounded sample per step."""
    if rank != 0:
        return
    n, B, delta, dt = workload(args.config, args.batch, args.n)
    import oracle
    from paper_1802_01359_b200 import signals

    ncores = oracle.num_threads()
    if args.config == "cfg3":
        # one 2^26 signal is out of the literal iteration's reach: each step is the paper's direct form
        # (oracle/direct_form.py) on a 2^20-sample cfg3-recipe signal
        from oracle import direct_form as dfo

        S, m = 1, 1 << 20
        s = signals.cfg3_signal(0, n=m)
        for _ in range(min(args.warmup, 1)):
            dfo.decompose(s, delta=delta)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            dfo.decompose(s, delta=delta)
        dt_s = (time.perf_counter() - t0) / args.steps
        value = m / dt_s
        line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt_s * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"cfg3 recipe, one n=2^20 signal per step (bounded sample of the n={n} signal)",
                           "n": m, "xi": 1.6, "delta": delta, "max_inner": 200, "max_imfs": 10},
                "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                                 "sample": "oracle/direct_form.py on one 2^20 cfg3-recipe signal per step"},
                "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    S = max(ncores, 16) if n <= 8192 else ncores  # signals per step (bounded sample of the batch)
    if args.config == "cfg2":  # ~3e11 FMAs per signal for the literal iteration: the direct form, 8 signals a step
        from oracle import direct_form as dfo

        S, ncores = 8, 1
        s = signals.make_batch("cfg2", batch=S)
        for _ in range(min(args.warmup, 1)):
            dfo.decompose(s[0], delta=delta)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            for b in range(S):
                dfo.decompose(s[b], delta=delta)
        step_s = (time.perf_counter() - t0) / args.steps
    else:
        s = signals.make_batch(args.config, batch=S, n=n if args.config == "cfg4" else None).astype(np.float64)
        for _ in range(args.warmup):
            oracle.decompose(s[: max(1, ncores)], delta=delta)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            oracle.decompose(s, delta=delta)
        step_s = (time.perf_counter() - t0) / args.steps
    value = S * n / step_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": {"workload": f"{args.config}: {S}-signal sample of the {B}x{n} {dt} batch per step",
                       "n": n, "batch_per_step": S, "xi": 1.6, "delta": delta, "max_inner": 200, "max_imfs": 10},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ncores, "kind": "oracle",
                             "sample": f"{S} signals of {args.config} per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import copy

    import torch

    line = run_ours(args, world, rank, local)
    if args.config == "cfg1" and args.batch is None and not args.no_secondary:
        # BASELINE.json's other batched fp64 workload, config 2 (512 x 65536, the streamed regime), timed in the
        # same run by the same contract (weak scaling per rank) and reported beside the headline line
        a2 = copy.copy(args)
        a2.config, a2.steps = "cfg2", max(1, min(args.steps, 5))
        l2 = run_ours(a2, world, rank, local)
        if line is not None and l2 is not None:
            line["secondary"] = {"cfg2": {k: l2[k] for k in ("value", "unit", "ms_per_step", "steps", "warmup",
                                                             "dtype", "config", "roofline", "cpu_baseline", "e2e",
                                                             "gpu_launches", "clocks")}}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_ours(args, world, rank, local):
    """One timed workload (args.config) through the public C ABI; returns the JSON line on rank 0, else None."""
    import torch

    torch.cuda.set_device(local)
    from paper_1802_01359_b200 import fif, signals

    n, B, delta, dt = workload(args.config, args.batch, args.n)
    scaling, parallelism = "weak", f"batch split x{world}, no collective"
    if args.config == "cfg3":
        # one long signal: strong scaling over the ranks (time-block shards, NCCL exchange steps)
        full = signals.cfg3_signal(0, n=n)
        if world > 1:
            plan = fif.Plan.dist(n, rank, world, uid=share_uid(rank, fif.nccl_unique_id), delta=delta)
            s_host = time_block(full, rank, world)
            parallelism = f"distributed x{world}: time-block shards, NCCL all-to-all + all-gather per IMF"
        elif args.emulate > 1:
            plan = fif.Plan.dist(n, 0, args.emulate, delta=delta, emulated=True)
            s_host = np.ascontiguousarray(full.reshape(args.emulate, n // args.emulate))
            parallelism = f"distributed algorithm, {args.emulate} ranks emulated on 1 GPU"
        else:
            plan = fif.Plan(n, 1, dt, delta=delta)
            s_host = full[None]
            parallelism = "single GPU, streamed regime"
        scaling = "strong"
        del full
    else:
        s_host = signals.make_batch(args.config, batch=B, start=rank_start(rank, B),
                                    n=n if args.config == "cfg4" else None)
        plan = fif.Plan(n, B, dt, delta=delta)
    # the eigenvalues of every scaling L precomputed once per plan (outside the timed region,
    # like the FFT twiddles); bit-identical decomposition (tests/test_gpu_options.py)
    eig = plan.launch_config()["regime"] == "resident" and not args.no_eig
    if eig:
        plan.set_eigen_table(True)
    x = torch.from_numpy(s_host).cuda()
    imfs, count, lens, iters = plan.alloc_outputs()
    stream = torch.cuda.current_stream()
    cfgl = plan.launch_config()

    for _ in range(max(args.warmup, 3)):
        plan.decompose(x, imfs, count, lens, iters, stream=stream)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        plan.decompose(x, imfs, count, lens, iters, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    clk = clocks.stop()
    ms = max_over_ranks(ms, world, "cuda")

    # roofline (dominant kernel = the single resident kernel: its launch duration = the step)
    cnt = count.cpu().numpy()
    if cfgl["regime"] == "distributed":
        cnt = cnt[:1]  # one signal; the count is replicated on every (emulated) rank
    Mtot = int(np.clip(cnt, 0, None).sum())
    eb = 8 if dt == "f64" else 4
    # on-chip regimes (resident, cluster): one read+write pass per transform; four-step (streamed, distributed): two
    passes = 2 if cfgl["regime"] in ("resident", "cluster") else 4
    fft_bytes = passes * n * eb * (Mtot + B)      # passes*n*b per transform, (M+1) transforms per signal
    comp_bytes = n * eb * (Mtot + 2 * B)          # read s once + write M IMFs + trend
    written_bytes = n * eb * B * (plan.max_imfs + 1) + n * eb * B  # output slots + input
    if args.config == "cfg3" and world > 1:       # per-GPU roofline: this rank's share of the bytes
        fft_bytes, comp_bytes, written_bytes = fft_bytes // world, comp_bytes // world, written_bytes // world
    peak, peak_kind = hbm_peak()
    ach = fft_bytes / (ms * 1e-3) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic_r01.json")
    if os.path.exists(tpath) and args.config == "cfg1" and args.batch is None:
        try:
            traffic = json.load(open(tpath)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    samples = n if args.config == "cfg3" else B * n * world
    value = samples / (ms * 1e-3)

    # e2e through the public host API (pinned host buffers; H2D + kernels + D2H inside the timed region)
    e2e = None
    if not args.no_e2e and cfgl["regime"] == "distributed":
        # e2e through fif_decompose with this rank's block copied in from pinned host memory and its
        # IMF block + integers copied back, inside the timed region
        hs = torch.from_numpy(s_host).pin_memory()
        h_out = [torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory() for t in (imfs, count, lens, iters)]
        ksteps = max(1, min(args.steps, 3))
        barrier()
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for _ in range(ksteps):
            x.copy_(hs, non_blocking=True)
            plan.decompose(x, imfs, count, lens, iters, stream=stream)
            for h, d in zip(h_out, (imfs, count, lens, iters)):
                h.copy_(d, non_blocking=True)
        e3.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e2.elapsed_time(e3) / ksteps, world, "cuda")
        e2e = {"value": samples / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": hs.numel() * hs.element_size(),
               "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in h_out), "ms_per_step": ems,
               "steps": ksteps, "path": "fif_decompose + cudaMemcpyAsync from/to pinned host (per rank)"}
    elif not args.no_e2e:
        hs = torch.from_numpy(s_host).pin_memory()
        h_out = [torch.empty(tuple(t.shape), dtype=t.dtype).pin_memory() for t in (imfs, count, lens, iters)]
        plan.decompose_host(hs, *h_out, stream=stream)  # warm-up (allocates staging)
        ksteps = max(1, min(args.steps, 3))
        barrier()
        torch.cuda.synchronize()
        e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2.record(stream)
        for _ in range(ksteps):
            plan.decompose_host(hs, *h_out, stream=stream)
        e3.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e2.elapsed_time(e3) / ksteps, world, "cuda")
        h2d = hs.numel() * hs.element_size()
        d2h = sum(t.numel() * t.element_size() for t in h_out)
        e2e = {"value": samples / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems, "steps": ksteps}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, n, delta, n4=n if args.config == "cfg4" else None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": dt, "data": "synthetic",
            "config": {"workload": (f"{args.config}: one signal of n={n} {dt} over {world} GPU(s) (BASELINE.json "
                                    f"configs[3])") if args.config == "cfg3" else
                                   (f"{args.config}: {B} signals x n={n} {dt} per GPU (BASELINE.json configs"
                                    f"[{args.config[-1]}])"),
                       "n": n, "batch_per_gpu": B, "xi": 1.6, "delta": delta, "max_inner": 200, "max_imfs": 10,
                       "window": "tri_sq (R1)", "parallelism": parallelism, "regime": cfgl["regime"],
                       "eigen_table": eig,
                       "l2": f"inputs+outputs {written_bytes / 1e9:.2f} GB/step > 126 MB L2 (no flush needed)",
                       "imfs_per_signal_mean": Mtot / B, "launch": cfgl},
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                         "traffic": traffic, "peak_kind": peak_kind,
                         "model": f"FFT-pass bytes {passes}*n*{eb}*(M+1) per signal (SURVEY.md 8d)",
                         "scope": "the single resident kernel" if cfgl["regime"] == "resident" else
                                  ("the single cluster kernel" if cfgl["regime"] == "cluster" else "whole step"),
                         "compulsory_frac": comp_bytes / (ms * 1e-3) / 1e9 / peak,
                         "written_bytes_per_launch": written_bytes},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * cfgl["kernels_per_call"],
            "clocks": clk,
        }
    plan.close()
    return line if rank == 0 else None


if __name__ == "__main__":
    main()
