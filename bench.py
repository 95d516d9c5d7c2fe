#!/usr/bin/env python
"""Benchmark of the batched verification step (CoSine, arXiv 2503.10325) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl reference]

One "step" = one cosine_verify_batch call over one batch of synthetic inputs already
resident in HBM (all of SURVEY §8(a): target softmax stats, drafter normalisers,
Eq. 4 fusion, acceptance, first rejection, residual / bonus resample).  For N > 1
(one process per GPU; `--gpus N` re-launches itself under torch.distributed.run when
WORLD_SIZE is unset) every rank verifies its own batch of the same shape with distinct
global request ids: weak scaling, no data-path collective (requests are independent,
Alg. 2).  c5 is the vocabulary-sharded call (strong scaling).  Prints ONE JSON
line on rank 0.

`--impl reference` times the CPU oracle (oracle/, fp64 C) on the host cores as the
reference arm: each step verifies a bounded sample of the workload's requests, one
request slice per host thread.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "verified draft tokens/sec and HBM GB/s vs 8 TB/s at 1/2/4/8 B200"
UNIT = "verified draft tokens/s"
WORKLOADS = {
    "c1": "c1: batch=1, 2 drafters, k=4, vocab=32000, fp32 logits/probs, T=1",
    "c2": "c2: batch=64, 3 drafters, k=8, vocab=32000 (Llama-2), bf16 logits/probs, T=1",
    "c3": "c3: batch=256, 4 drafters, k=8, vocab=128256 (Llama-3), bf16 logits/probs, T=1",
    "c4": "c4: tree-shaped drafts, 64-node tree per request (schedule 4,2,2,1,1,1,1,1), batch=128, "
          "4 drafters, vocab=128256, bf16, T=1",
    "c5": "c5: batch=1024, 4 drafters, k=8, vocab=128256 (Llama-3) split in N column shards (tensor-parallel "
          "LM head layout), bf16, T=1, vocabulary-sharded verification over NCCL",
}
WEIGHTS = {"conf": 0, "winner": 1, "uniform": 2, "point": 3}
SELECTS = {"argmax": 0, "sample": 1}
L2_BYTES = 126 * 2**20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--weights", default="conf", choices=sorted(WEIGHTS),
                    help="fusion weights (Eq. 4 CONF default; reading #2)")
    ap.add_argument("--select", default="argmax", choices=sorted(SELECTS),
                    help="argmax = Eq. 4 fused token (paper-literal); sample = x* ~ fused q (reading #3)")
    ap.add_argument("--cluster-size", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-threads", type=int, default=0, help="oracle threads (0 = all host cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--flush", default="auto", choices=["auto", "on", "off"],
                    help="flush L2 between timed calls (auto: when the inputs are < 4x L2)")
    ap.add_argument("--traffic", default="auto", choices=["auto", "off"],
                    help="auto: measure the kernel's DRAM bytes with an ncu child run (N = 1 only)")
    ap.add_argument("--lazy", action="store_true",
                    help="early-exit verification (cosine_verify_batch_lazy, SURVEY 8(f) NEXT-1)")
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl"],
                    help="c5: in-kernel NVLink peer writes when available (auto) or NCCL all-gathers")
    ap.add_argument("--watchdog", type=float, default=0.0,
                    help="dump every thread's stack and exit after this many seconds (0 = off)")
    a = ap.parse_args()
    if a.lazy and a.config == "c5":
        ap.error("--lazy runs on unsharded contexts (c1..c4)")
    if a.config in ("c4", "c5") and a.select != "argmax":
        ap.error("tree / vocabulary-sharded verification takes ARGMAX selection")
    if a.lazy and a.select != "argmax":
        ap.error("lazy verification takes ARGMAX selection")
    return a


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch_ranks(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, one rank
    per GPU; inside torchrun: the world size must equal --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if int(world or 1) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler(threading.Thread):
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    def __init__(self, device_index: int, period: float = 0.01):
        super().__init__(daemon=True)
        self.period = period
        self.samples = []
        self.reasons = set()
        self.stop_ev = threading.Event()
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    def run(self):
        if not self.ok:
            return
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
            "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
            "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
            "display_clock_setting": 0x100,
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in names.items():
                    if r & bit and n != "gpu_idle":
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(self.period)

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cfg_of(name):
    import synth
    return dict(synth.CONFIGS[name])


def cpu_threads(args):
    return args.cpu_threads if args.cpu_threads > 0 else (os.cpu_count() or 1)


# --------------------------------------------------------------------------------------
def cpu_oracle_rate(host_inputs, k, V, budget_s, seed, threads, wm=0, sm=0):
    """The CPU oracle as it stands, on `threads` host threads (one request per thread at a time,
    GIL released in the C code), over rounds of `threads` whole requests of the workload — the
    sample cycled — until ~budget_s seconds; returns (tokens/s, requests, seconds)."""
    import oracle
    B = host_inputs["target"].shape[0]
    done_req, spent, b0 = 0, 0.0, 0
    while spent < budget_s:
        b1 = min(B, b0 + threads)
        t0 = time.perf_counter()
        oracle.verify_batch_parallel(host_inputs["target"][b0:b1], host_inputs["draft"][b0:b1],
                                     host_inputs["draft_tokens"][b0:b1], host_inputs["request_ids"][b0:b1],
                                     threads=threads, temperature=1.0, seed=seed, vocab=V, weight_mode=wm,
                                     select_mode=sm)
        spent += time.perf_counter() - t0
        done_req += b1 - b0
        b0 = 0 if b1 >= B else b1
    return done_req * k / spent, done_req, spent


def run_reference(args):
    """Reference arm: the CPU oracle on the box's host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    import oracle
    c = cfg_of(args.config)
    B, N, k, V, dt = c["B"], c["N"], c["k"], c["V"], c["dtype"]
    threads = cpu_threads(args)
    steps, warm = args.steps, args.warmup
    per = min(B, threads)  # requests per step: one per thread (a bounded sample of the batch)
    # bound the whole run to a few minutes of host time (~30 ms per c3-sized request and thread)
    est = 0.03 * (V / 128256) * (k + 1 + k * N) / 41 * (warm + steps)
    if est > 150:
        steps = max(3, int(steps * 150 / est))
    nreq = min(B, per * 4)
    inp = synth.linear_inputs(nreq, k, N, V, dtype=dt, seed=args.seed, device="cpu", chunk=4)
    times = []
    for s in range(warm + steps):
        b0 = (s * per) % nreq
        sl = slice(b0, b0 + per)
        t0 = time.perf_counter()
        oracle.verify_batch_parallel(inp["target"][sl], inp["draft"][sl], inp["draft_tokens"][sl],
                                     inp["request_ids"][sl], threads=threads, temperature=1.0, seed=args.seed,
                                     vocab=V, weight_mode=WEIGHTS[args.weights], select_mode=SELECTS[args.select])
        if s >= warm:
            times.append(time.perf_counter() - t0)
    total = sum(times)
    value = steps * per * k / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * total / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.config], "weights": args.weights, "select": args.select,
                   "sample_per_step": f"{per} requests ({per * k} verified tokens), one per host thread"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": f"{steps} steps x {per} requests of {args.config} (fp64 C oracle, "
                                   f"{threads} threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_traffic(args, kernel_regex):
    """DRAM bytes (read + write) and duration of one launch of the dominant kernel, from an ncu
    child run of this script (its own numbers are not used; N = 1 only)."""
    ncu = "/usr/local/cuda/bin/ncu"
    if not os.path.exists(ncu):
        return None, "ncu not found"
    cmd = [ncu, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "-k", f"regex:{kernel_regex}", "-s", "3", "-c", "1", "--csv",
           sys.executable, os.path.abspath(__file__), "--config", args.config, "--steps", "1", "--warmup", "3",
           "--weights", args.weights, "--select", args.select, "--no-cpu-baseline", "--no-e2e",
           "--traffic", "off", "--flush", "off"] + (["--lazy"] if args.lazy else [])
    try:
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    except Exception as e:  # pragma: no cover
        return None, f"ncu failed: {e}"
    vals = {}
    import csv
    import io
    rows = [ln for ln in res.stdout.splitlines() if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("\n".join(rows))):
        name, unit, v = r.get("Metric Name"), r.get("Metric Unit"), r.get("Metric Value", "").replace(",", "")
        try:
            x = float(v)
        except ValueError:
            continue
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3}.get(unit, 1)
        vals[name] = x * scale
    if "dram__bytes_read.sum" not in vals:
        return None, f"ncu gave no metrics (rc {res.returncode})"
    return vals, "ncu dram__bytes_read.sum + dram__bytes_write.sum, one launch (cold L2)"


# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    import paper_2503_10325_b200 as cv
    import synth
    from paper_2503_10325_b200 import sharding

    c = cfg_of(args.config)
    B, N, k, V, dt = c["B"], c["N"], c["k"], c["V"], c["dtype"]
    esz = torch.tensor([], dtype=dt).element_size()
    dev = torch.device("cuda", local)
    if args.config == "c4":
        return run_tree(args, c, dev, world, rank, local)
    if args.config == "c5":
        return run_vocab(args, c, dev, world, rank, local)
    wm, sm = WEIGHTS[args.weights], SELECTS[args.select]
    rids = sharding.weak_request_ids(B, rank)  # weak scaling: a full batch per rank, global ids
    inp = synth.linear_inputs(B, k, N, V, dtype=dt, seed=args.seed + 7919 * rank, device=dev,
                              rid_base=rids.start)
    ver = cv.Verifier(V, max_batch=B, k=k, N=N, device=local, target_dtype=dt, draft_dtype=dt,
                      seed=args.seed, cluster_size=args.cluster_size)
    stream = torch.cuda.current_stream(dev)
    alg_bytes = synth.algorithmic_bytes(B, k, N, V, esz, esz)
    flush = args.flush == "on" or (args.flush == "auto" and alg_bytes < 4 * L2_BYTES)
    # read (not write) 2x L2 between timed calls: the inputs are evicted and L2 holds only clean
    # lines, so the timed call pays no write-back of a memset's dirty lines
    scratch = torch.ones(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def step():
        ver.verify(inp["target"], inp["draft"], inp["draft_tokens"], inp["request_ids"],
                   temperature=1.0, lazy=args.lazy, weight_mode=wm, select_mode=sm)
        return cv.cosine_last_launch_count(ver.ctx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches = 0
    t_start.record(stream)
    for s in range(args.steps):
        if flush:
            scratch.sum()  # evict the inputs from L2 (untimed: outside this call's events)
        ev[s][0].record(stream)
        launches += step()
        ev[s][1].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler.stop_ev.set()
    sampler.join()
    kern_ms = [a.elapsed_time(b) for a, b in ev]
    elapsed_ms = sum(kern_ms) if flush else t_start.elapsed_time(t_end)
    # second timed pass with CUDA events recorded by the library around its dominant launch on
    # the launching stream (cosine_profile_*)
    cv.cosine_profile_enable(ver.ctx, True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for s in range(args.steps):
        if flush:
            scratch.sum()
        step()
    torch.cuda.synchronize()
    prof_ms, prof_n = cv.cosine_profile_read(ver.ctx)
    cv.cosine_profile_enable(ver.ctx, False)
    kernel_name = "cosine::stats_kernel (streams every input byte once; 1 of the call's 3 launches)"
    kernel_regex = "stats_kernel"
    if args.lazy:  # no single dominant launch: the whole call against its realised bytes
        # rows read per request: target 0..L, drafters at positions 0..min(L, k-1) — the round
        # holding L (kLazySpan = 2 positions per round) also streamed its other position — and
        # the final draw's rows (1 + N at a rejection, the bonus row otherwise)
        span = 2
        Ls = ver.accept_len[:B].long().clamp_min(0)
        span_end = torch.clamp((Ls // span) * span + span, max=k + 1)  # positions 0 .. span_end - 1 read
        rows = span_end + torch.clamp(span_end, max=k) * N + torch.where(Ls < k, 1 + N, 1)
        alg_bytes = int(rows.sum()) * V * esz
        prof_ms, prof_n = statistics.mean(kern_ms), 1
        kernel_name, kernel_regex = "whole lazy call (rounds of stats + lazy_decide, then resample)", "stats_kernel"
    elapsed_ms = sharding.max_over_ranks(elapsed_ms, device=dev)  # the slowest rank's device time
    acc = ver.accept_len[:B].float().mean().item()
    status_nonzero = int((ver.status[:B] & 0xff).ne(0).sum().item())

    tokens_per_step = B * k * world
    value = tokens_per_step * args.steps / (elapsed_ms / 1e3)
    step_avg_s = statistics.mean(kern_ms) / 1e3
    kern_avg_s = (prof_ms / max(prof_n, 1)) / 1e3
    achieved = alg_bytes / kern_avg_s / 1e9
    peak, peak_src = peaks()

    # ---- e2e: the public call from pinned host buffers, H2D + kernel + D2H in the region
    e2e = None
    if not args.no_e2e:
        names = ("target", "draft", "draft_tokens", "request_ids")
        host = {n: inp[n].cpu().pin_memory() for n in names}
        devbuf = {n: torch.empty_like(inp[n]) for n in names}
        h2d = sum(host[n].numel() * host[n].element_size() for n in names)
        d2h = B * 4 + B * (k + 1) * 4 + B * 4
        ver.verify_host(host, devbuf, weight_mode=wm, select_mode=sm)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            ver.verify_host(host, devbuf, weight_mode=wm, select_mode=sm)
        e1.record(stream)
        torch.cuda.synchronize()
        te = sharding.max_over_ranks(e0.elapsed_time(e1), device=dev)
        e2e = {"value": tokens_per_step * args.e2e_steps / (te / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": te / args.e2e_steps}
        del devbuf, host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads(args)
        host_inp = {n: inp[n][: min(B, 4 * threads)].cpu() for n in ("target", "draft", "draft_tokens", "request_ids")}
        rate, nreq, spent = cpu_oracle_rate(host_inp, k, V, args.cpu_seconds, args.seed, threads, wm, sm)
        rate1, nreq1, spent1 = cpu_oracle_rate(host_inp, k, V, args.cpu_seconds / 3, args.seed, 1, wm, sm)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"{nreq} requests of {args.config} ({nreq * k} verified tokens; the first "
                         f"{host_inp['target'].shape[0]} of the batch, cycled), fp64 C oracle, {threads} threads "
                         f"(one request per thread at a time), {spent:.1f} s",
               "single_thread": {"value": rate1, "cores": 1, "sample": f"{nreq1} requests, {spent1:.1f} s"}}
    ver.close()
    del inp
    traffic, traffic_src = None, "not measured"
    if rank == 0 and world == 1 and args.traffic == "auto":
        torch.cuda.empty_cache()
        t, traffic_src = ncu_traffic(args, kernel_regex)
        if t is not None:
            traffic = t["dram__bytes_read.sum"] + t.get("dram__bytes_write.sum", 0.0)

    if rank == 0:
        clocks = sampler.result()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16" if dt == torch.bfloat16 else "f32",
            "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config] + (" — LAZY early-exit verification (NEXT-1): rows after "
                                                              "the first rejection are not read; bytes = realised"
                                                              if args.lazy else ""),
                       "weights": args.weights, "select": args.select,
                       "batch_per_gpu": B, "global_batch": B * world,
                       "k": k, "drafters": N, "vocab": V, "parallelism": f"batch-sharded x{world}",
                       "l2": (f"L2 flushed between timed calls (a {2 * L2_BYTES >> 20} MiB read, outside the "
                              f"timed events; inputs {alg_bytes / 1e6:.1f} MB)") if flush else
                             f"inputs {alg_bytes / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)",
                       "mean_accept_len": acc, "request_errors": status_nonzero},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src,
                         "frac_of_8tbs": achieved / 8000.0, "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel_us": kern_avg_s * 1e6, "kernel": kernel_name,
                         "kernel_launches_timed": prof_n,
                         "step_us": step_avg_s * 1e6, "step_achieved": alg_bytes / step_avg_s / 1e9,
                         "step_frac": alg_bytes / step_avg_s / 1e9 / peak,
                         "step_frac_of_8tbs": alg_bytes / step_avg_s / 1e9 / 8000.0},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_tree(args, c, dev, world, rank, local):
    """c4: one cosine_verify_tree call per step; verified draft tokens = B x 64."""
    import torch
    import torch.distributed as dist
    import paper_2503_10325_b200 as cv
    import synth
    from paper_2503_10325_b200 import sharding
    B, N, V, dt = c["B"], c["N"], c["V"], c["dtype"]
    t = synth.tree_inputs(B, N, V, dtype=dt, seed=args.seed + 7919 * rank, device=dev,
                          rid_base=sharding.weak_request_ids(B, rank).start)
    nn, I = t["J"] + 1, t["I"]
    esz = torch.tensor([], dtype=dt).element_size()
    ctx = cv.cosine_verify_init(V, device=local, max_batch=B, max_draft_len=1, max_drafters=N, seed=args.seed,
                                target_dtype=dt, draft_dtype=dt, max_tree_nodes=nn)
    al = torch.empty(B, dtype=torch.int32, device=dev)
    an = torch.empty(B, nn, dtype=torch.int32, device=dev)
    ot = torch.empty(B, nn, dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    wm = WEIGHTS[args.weights]

    def step():
        cv.cosine_verify_tree(ctx, t["parent"], t["node_token"], t["internal_row"], t["target"], t["draft"],
                              t["node_draft_tokens"], t["request_ids"], al, an, ot, st, temperature=1.0,
                              lazy=args.lazy, weight_mode=wm)
        return cv.cosine_last_launch_count(ctx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for _ in range(args.steps):
        launches += step()
    e1.record(stream)
    torch.cuda.synchronize()
    sampler.stop_ev.set()
    sampler.join()
    ms = sharding.max_over_ranks(e0.elapsed_time(e1), device=dev) / args.steps
    tokens = B * t["J"] * world
    alg = synth.tree_algorithmic_bytes(B, nn, I, N, V, esz, esz)
    accounting = "all nodes read once (whole call)"
    emitted = (al.clamp_min(0) + 1).sum().item() * world
    if args.lazy:  # realised path bytes: the visited nodes' rows + one pass per rejection / bonus
        par = t["parent"][0].tolist()
        irow = t["internal_row"][0].tolist()
        kids = {j: [c for c in range(1, nn) if par[c] == j] for j in range(nn)}
        rows = 0
        for b in range(B):
            path = [0] + [int(x) for x in an[b].tolist() if x >= 0]
            for d, j in enumerate(path):
                node_rows = 1 + (N if irow[j] >= 0 else 0)
                passes = 1  # the node's statistics
                if d + 1 < len(path):
                    passes += kids[j].index(path[d + 1])  # children rejected before the accepted one
                else:
                    passes += len(kids[j]) if kids[j] else 1  # all children rejected, or the bonus pass
                rows += passes * node_rows
        alg = rows * V * esz
        accounting = "LAZY (NEXT-1): realised path bytes (visited nodes' statistics + rejection / bonus passes)"
    peak, peak_src = peaks()
    acc = al.float().mean().item()
    if rank == 0:
        line = {
            "metric": METRIC, "value": tokens / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOADS["c4"] + (" — LAZY walk (NEXT-1): only the visited nodes' rows are read"
                                                      if args.lazy else ""),
                       "weights": args.weights, "batch_per_gpu": B, "global_batch": B * world,
                       "tree_nodes": t["J"], "internal_nodes": I, "drafters": N, "vocab": V,
                       "parallelism": f"batch-sharded x{world}", "mean_accept_len": acc,
                       "emitted_tokens_per_s": emitted / (ms / 1e3),
                       "l2": f"inputs {alg / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"},
            "roofline": {"bound": "hbm", "achieved": alg / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / (ms / 1e3) / 1e9 / peak, "traffic": None, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg, "accounting": accounting,
                         "frac_of_8tbs": alg / (ms / 1e3) / 1e9 / 8000.0},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": sampler.result(),
        }
        print(json.dumps(line), flush=True)
    cv.cosine_verify_destroy(ctx)
    if world > 1:
        dist.destroy_process_group()


def run_vocab(args, c, dev, world, rank, local):
    """c5: the same B = 1024 requests on every rank, each rank holding 1/N of the vocabulary
    columns; one collective cosine_verify_batch per step (kernels + NCCL
    all-gathers).  Total work is fixed: strong scaling; value = B k / step time."""
    import torch
    import torch.distributed as dist
    import paper_2503_10325_b200 as cv
    import synth
    from paper_2503_10325_b200 import sharding
    B, N, k, V, dt = c["B"], c["N"], c["k"], c["V"], c["dtype"]
    esz = torch.tensor([], dtype=dt).element_size()
    vb, ve = sharding.vocab_shard(V, world, rank)
    W = ve - vb
    ld = (W + 7) // 8 * 8
    # the same global inputs on every rank (seeded), this rank's columns kept, generated in
    # request slices so that only one slice of the full rows exists at a time
    tgt = torch.empty(B, k + 1, ld, dtype=dt, device=dev)
    drf = torch.empty(B, k, N, ld, dtype=dt, device=dev)
    xs, rids = [], []
    sl = 64
    for b0 in range(0, B, sl):
        part = synth.linear_inputs(sl, k, N, V, dtype=dt, seed=args.seed + b0, device=dev, rid_base=b0)
        tgt[b0:b0 + sl, :, :W] = part["target"][..., vb:ve]
        drf[b0:b0 + sl, :, :, :W] = part["draft"][..., vb:ve]
        xs.append(part["draft_tokens"])
        rids.append(part["request_ids"])
        del part
    toks, rid = torch.cat(xs), torch.cat(rids)
    if world > 1:
        ctx = sharding.init_vocab_sharded(V, device=local, max_batch=B, max_draft_len=k, max_drafters=N,
                                          target_dtype=dt, draft_dtype=dt, seed=args.seed,
                                          exchange=1 if args.exchange == "nccl" else 0)
    else:
        ctx = cv.cosine_verify_init(V, device=local, max_batch=B, max_draft_len=k, max_drafters=N,
                                    target_dtype=dt, draft_dtype=dt, seed=args.seed)
    ver = cv.Verifier(V, max_batch=B, k=k, N=N, device=local, ctx=ctx)
    exchange = cv.cosine_exchange_mode(ver.ctx)
    stream = torch.cuda.current_stream(dev)
    wm = WEIGHTS[args.weights]

    def step():
        ver.verify(tgt, drf, toks, rid, temperature=1.0, weight_mode=wm)
        return cv.cosine_last_launch_count(ver.ctx)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.05)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for _ in range(args.steps):
        launches += step()
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler.stop_ev.set()
    sampler.join()
    ms = sharding.max_over_ranks(e0.elapsed_time(e1), device=dev) / args.steps
    cv.cosine_profile_enable(ver.ctx, True)
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    stats_ms, stats_n = cv.cosine_profile_read(ver.ctx)  # one bracketed stats launch per request slice
    cv.cosine_profile_enable(ver.ctx, False)
    kern_s = max(sharding.max_over_ranks(stats_ms / args.steps, device=dev) / 1e3, 1e-9)  # per call
    acc = ver.accept_len[:B].float().mean().item()
    errs = int((ver.status[:B] & 0xff).ne(0).sum().item())
    alg_rank = (B * (k + 1) * W * esz + B * k * N * W * esz + 4 * B * k * N + 8 * B)
    alg_total = synth.algorithmic_bytes(B, k, N, V, esz, esz)
    peak, peak_src = peaks()
    achieved = alg_rank / kern_s / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": B * k / (ms / 1e3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOADS["c5"], "weights": args.weights, "global_batch": B, "k": k,
                       "drafters": N, "vocab": V,
                       "shard_columns": W, "parallelism": f"vocab-sharded x{world}",
                       "exchange": exchange, "mean_accept_len": acc,
                       "request_errors": errs,
                       "l2": f"inputs {alg_rank / 1e9:.2f} GB per GPU > 126 MB L2 (no flush needed)"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                         "kernel": "cosine::stats_kernel (local columns; summed over the call's request slices)",
                         "kernel_us": kern_s * 1e6, "kernel_launches_per_call": stats_n / args.steps,
                         "algorithmic_bytes_per_launch": alg_rank, "algorithmic_bytes_total": alg_total,
                         "step_achieved_per_gpu": alg_rank / (ms / 1e3) / 1e9,
                         "step_frac": alg_rank / (ms / 1e3) / 1e9 / peak},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": sampler.result(),
        }
        print(json.dumps(line), flush=True)
    ver.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = parse()
    if a.watchdog > 0:
        import faulthandler
        faulthandler.dump_traceback_later(a.watchdog, exit=True)
    launch_ranks(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
