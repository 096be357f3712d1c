#!/usr/bin/env python
"""Benchmark: batched <H> + adjoint gradient circuits/s (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl tcx|reference] [--config I]

One step = one tcx_grad_batch over the rank's theta batch (every row: forward window
passes, lambda = H psi, adjoint backward passes, fp64 reductions) followed by the NCCL
all-reduce of the loss sum_b E_b and the batch-summed gradient (north_star: "final NCCL
all-reduce of loss and gradient").  Default workload: BASELINE configs[1] (n=20 Heisenberg
VQE, HEA depth 10, B=1024 theta per rank, complex64).  Scaling: weak (B per rank fixed).
For N > 1 launch with torchrun (one process per GPU, MASTER_ADDR=127.0.0.1).
`--impl reference` times the CPU oracle (oracle/, the tier's reference arm) on host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def load_peaks():
    try:
        with open(PEAKS) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# -------------------------------------------------------------- reference
def cpu_oracle_rows(circ, H, theta, threads, mode="grad"):
    from oracle import oracle as orc
    t0 = time.perf_counter()
    if mode == "grad":
        orc.value_grad_batch(circ, H, theta, nthreads=threads)
    else:
        orc.expect_batch(circ, H, theta, nthreads=threads)
    return time.perf_counter() - t0


def survey_flop_model(circ, H, B, ms_step, alu_peak):
    """SURVEY §8(d)'s ALU flop model for a whole <H>+grad step, beside the library's own
    per-kernel model: 6 flop/amp per rotation forward (structured 2x2), 0 for CNOT/CZ/SWAP,
    15 flop/amp per parameterised gate backward (U^dagger on psi and lambda + the
    Im<lambda|G|psi> term), 4 flop/amp per Pauli term for lambda = H psi.  Fraction = model
    flops / step time / the FP32 (FP64) FMA peak."""
    amps = float(1 << circ.n)
    rot = sum(1 for g in circ.gates if g.name in ("rx", "ry", "rz", "rxx", "ryy", "rzz", "u1", "rrot"))
    par = sum(1 for g in circ.gates if g.param >= 0)
    per_amp = 6.0 * rot + 15.0 * par + 4.0 * len(H.weights)
    fl = per_amp * amps * B
    ach = fl / (ms_step / 1e3)
    return {"flops_per_step": fl, "achieved_tflops": ach / 1e12, "peak_tflops": alu_peak / 1e12,
            "frac": ach / alu_peak,
            "model": "SURVEY 8(d): 6 flop/amp per rotation fwd, 15 per parameterised gate bwd, "
                     "4 per Pauli term; whole step (all kernels) / measured FMA peak"}


def host_cpu():
    """(logical cores, CPU model) of this host, recorded with every oracle figure."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count() or 1, model


def cpu_baseline(circ, H, theta, mode, name, max_rows=0):
    """SURVEY §8d oracle timing on this host: (i) one theta row on one thread, (ii) the same
    oracle with OpenMP over theta rows on every host core (one row per core).  Bounded
    samples of the workload (whole rows), linear in rows; cfg5's 2^33 state does not fit the
    oracle (closed-form pinned instead) and cfg4 has B = 1 (row-parallel OpenMP cannot use
    more than one core there), so those report the single-thread figure only."""
    nproc, model = host_cpu()
    if name.startswith("cfg4"):
        # B = 1 and 8,900 gates on 2^30 amplitudes: hours in the oracle.  Time one layer of the
        # same generator at n = 26 on one thread and scale linearly (the oracle's cost is gates x
        # amplitudes): x 2^(n-26) amplitudes x layers
        layers = 200
        c1 = W.random_deep_circuit(26, 1, 4)
        t1 = cpu_oracle_rows(c1, W.pauli_sum(26, [({0: "Z"}, 1.0)]), np.zeros((1, 0)), 1, "expect")
        est = t1 * (1 << (circ.n - 26)) * layers
        return {"value": 1.0 / est, "unit": "circuits/s", "cores": 1, "kind": "oracle",
                "nproc": nproc, "cpu_model": model,
                "sample": f"extrapolated: 1 layer of the cfg4 generator at n = 26 took {t1:.1f} s on one "
                          f"thread, x 2^{circ.n - 26} amplitudes x {layers} layers = {est:.0f} s per circuit "
                          "(B = 1: the oracle parallelises over rows only)"}
    if circ.n > 28:
        return {"value": None, "unit": "circuits/s", "cores": 0, "kind": "oracle",
                "nproc": nproc, "cpu_model": model,
                "sample": f"N/A: a {circ.n}-qubit state does not fit the float64 oracle"}
    t1 = cpu_oracle_rows(circ, H, theta[:1], 1, mode)
    single = {"value": 1.0 / t1, "cores": 1, "sample": f"1 theta row of {name}, {t1:.1f} s"}
    rows = min(nproc, theta.shape[0]) if not max_rows else min(nproc, theta.shape[0], max_rows)
    if rows <= 1:
        return {"value": single["value"], "unit": "circuits/s", "cores": 1, "kind": "oracle",
                "nproc": nproc, "cpu_model": model, "sample": single["sample"] +
                " (B = 1: the oracle parallelises over rows only)", "single_thread": single}
    tn = cpu_oracle_rows(circ, H, theta[:rows], rows, mode)
    return {"value": rows / tn, "unit": "circuits/s", "cores": rows, "kind": "oracle",
            "nproc": nproc, "cpu_model": model,
            "sample": f"{rows} theta rows of {name}, OpenMP one row per core, {tn:.1f} s",
            "single_thread": single}


def run_reference(args, rank, world):
    """The tier's reference arm: the CPU oracle, as it stands, on host cores."""
    if rank != 0:
        return 0
    name, circ, H, theta, dtype = W.config(args.config, B=args.batch)
    mode = args.mode or ("expect" if circ.n_params == 0 else "grad")
    cores, model = host_cpu()
    rows = max(1, min(cores, args.ref_rows or cores, theta.shape[0]))
    sample = theta[:rows]
    for _ in range(args.warmup):
        cpu_oracle_rows(circ, H, sample[:1], 1, mode)
    total = 0.0
    for _ in range(args.steps):
        total += cpu_oracle_rows(circ, H, sample, rows, mode)
    value = rows * args.steps / total
    unit = "circuits/s"
    line = {
        "metric": ("batched <H>+grad circuits/s (%s)" if mode == "grad" else
                   "batched <H> circuits/s (%s, forward only)") % name, "value": value, "unit": unit,
        "impl": "reference", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": name, "global_batch": rows, "seq_len": None,
                   "parallelism": "oracle: OpenMP over theta rows"},
        "cpu_baseline": {"value": value, "unit": unit, "cores": rows, "kind": "oracle",
                         "nproc": cores, "cpu_model": model,
                         "sample": f"{rows} theta rows of {name} per step (OpenMP, one per core)"},
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tcx", choices=["tcx", "reference"])
    ap.add_argument("--config", type=int, default=1,
                    help="BASELINE.json configs index (5: the paper's Table VII barren-plateau task)")
    ap.add_argument("--batch", type=int, default=None, help="theta rows per rank")
    ap.add_argument("--qubits", type=int, default=None,
                    help="override the config's qubit count (e.g. config 1 at n = 14..17 with --cluster-bits)")
    ap.add_argument("--cluster-bits", type=int, default=0,
                    help="cluster-resident states (SURVEY §8f f1): 2^g CTAs per theta row")
    ap.add_argument("--batch-qubits", type=int, default=None,
                    help="config 4: local qubits per rank (default 33)")
    ap.add_argument("--tile-bits", type=int, default=0)
    ap.add_argument("--coalesce-bits", type=int, default=0)
    ap.add_argument("--reg-bits", type=int, default=0)
    ap.add_argument("--max-ops-per-pass", type=int, default=0)
    ap.add_argument("--l2-rows", type=int, default=0,
                    help="theta rows per L2-resident group (-1 auto; 0 off)")
    ap.add_argument("--dtype", default=None, choices=["c64", "c128"],
                    help="override the config's state dtype (studies; e.g. cfg4 at complex64)")
    ap.add_argument("--dense-k", type=int, default=0,
                    help="fuse gates into dense k-qubit blocks (k = 1..5; cfg4 k-sweep)")
    ap.add_argument("--jit", type=int, default=1, help="1: per-circuit specialised kernels")
    ap.add_argument("--mode", default=None, choices=["grad", "expect"],
                    help="grad (E + adjoint gradient, default) or expect (forward + E only; cfg4)")
    ap.add_argument("--graph", type=int, default=-1,
                    help="1: capture one step (library kernels + all-reduce) in a CUDA graph and "
                         "replay it; 0: eager launches; -1 (default): graph only for launch-bound "
                         "steps (< 2 ms eager), so long steps keep per-kernel events in the timed region")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=0, help="reference arm rows (0: one per host core)")
    ap.add_argument("--virtual-ranks", type=int, default=1,
                    help="config 4 on one GPU: shard the state over this many virtual ranks")
    ap.add_argument("--cpu-rows", type=int, default=0, help="cpu_baseline rows (0: one per host core)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "tcx" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2205_10091_b200 import tcx

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=dev)

    if args.config == 4 and (world > 1 or args.virtual_ranks > 1):
        return run_sharded(args, world, rank, local, dev)

    name, circ, H, theta, dtype = W.config(args.config, B=args.batch, n=args.qubits)
    if args.qubits:
        name = name.replace(f"{W.config(args.config, B=1)[1].n}_", f"{args.qubits}_", 1)
    if args.dtype and args.dtype != dtype:
        name, dtype = name.replace("_" + dtype, "_" + args.dtype), args.dtype
    B = theta.shape[0]
    if world > 1 and rank > 0 and args.config in (0, 1, 2):  # distinct seeded rows per rank
        theta = W.thetas(B, circ.n_params, 1000 + rank) if args.config != 2 else \
            W.qaoa_thetas(B, 5, 1000 + rank)
    C = tcx.Circuit(circ, dtype, tile_bits=args.tile_bits, coalesce_bits=args.coalesce_bits,
                    reg_bits=args.reg_bits,
                    max_ops_per_pass=args.max_ops_per_pass,
                    jit=bool(args.jit), dense_k=args.dense_k, l2_rows=args.l2_rows,
                    cluster_bits=args.cluster_bits)
    P = tcx.Pauli(H)
    t_jit = time.perf_counter()
    mode = args.mode or ("expect" if circ.n_params == 0 else "grad")
    C.compile(P, B=B, kind=mode)  # the K.jit analog: excluded from timings
    t_jit = time.perf_counter() - t_jit
    info = C.info(P)
    th = torch.as_tensor(np.ascontiguousarray(theta)).to(dev)
    E = torch.empty(B, dtype=torch.float64, device=dev)
    G = torch.empty(B, max(circ.n_params, 1), dtype=torch.float64, device=dev)
    red = torch.empty(1 + circ.n_params, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    ws = tcx.Workspace()

    from paper_2205_10091_b200.dist import allreduce_loss_grad

    def step():
        if mode == "grad":
            tcx.grad_batch(C, P, th, stream=stream, ws=ws, out=(E, G))
            allreduce_loss_grad(E, G[:, :circ.n_params], out=red)
        else:
            Ex = tcx.expect_batch(C, P, th, stream=stream, ws=ws)
            allreduce_loss_grad(Ex, G[:, :0], out=red[:1])

    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(args.warmup):
        if i == args.warmup - 1:
            w0.record(stream)
        step()
    w1.record(stream)
    torch.cuda.synchronize(dev)
    use_graph = args.graph == 1 or (args.graph == -1 and w0.elapsed_time(w1) < 2.0)
    # CUDA graph of one step (streams and graphs instead of a tracing compiler): the
    # library's launches are plain stream work once its JIT modules and tables exist
    graph, graph_note = None, "eager"
    # single-process only: a captured NCCL collective that fails to instantiate could leave
    # the communicator unusable mid-run, and multi-GPU steps are not launch-bound
    if use_graph and world == 1:
        try:
            gs = torch.cuda.Stream(dev)
            gs.wait_stream(stream)
            with torch.cuda.stream(gs):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=gs):
                    step_on = stream
                    stream = gs
                    step()
                    stream = step_on
            torch.cuda.synchronize(dev)
            graph, graph_note = g, "cuda graph replay"
        except Exception as ex:  # capture unsupported here: time eager launches
            graph, graph_note = None, f"eager (graph capture failed: {type(ex).__name__})"
            torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if graph is None:  # per-kernel CUDA events live inside the timed region
        tcx.profile_enable(True)
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    prof_steps = args.steps
    if graph is not None:  # graph replays carry no per-kernel events: one extra eager step
        tcx.profile_enable(True)
        step()
        torch.cuda.synchronize(dev)
        prof_steps = 1
    tcx.profile_enable(False)
    prof = tcx.profile_read()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B * args.steps / (ms / 1e3)

    # ---- end to end through the host-buffer public API (pinned host memory); the
    # device-resident run's workspace is released first (cfg5's 128 GiB psi + lambda fits once)
    used_graph, graph = graph is not None, None
    ws.clear()
    torch.cuda.synchronize(dev)
    torch.cuda.empty_cache()
    th_h = torch.as_tensor(np.ascontiguousarray(theta)).pin_memory()
    E_h = torch.empty(B, dtype=torch.float64).pin_memory()
    G_h = torch.empty(B, max(circ.n_params, 1), dtype=torch.float64).pin_memory()
    ws2 = tcx.Workspace()

    def e2e_step():
        if mode == "grad":
            tcx.grad_batch_host(C, P, th_h.numpy(), E_h.numpy(), G_h.numpy(), stream=stream,
                                ws=ws2, device=dev)
        else:
            tcx.expect_batch_host(C, P, th_h.numpy(), E_h.numpy(), stream=stream, ws=ws2,
                                  device=dev)
    e2e_step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = world * B * args.steps / float(e2e_s.item())

    # ---- roofline of the dominant kernel class
    peaks, peak_src = load_peaks()
    by = {}
    for ph, idx, kms, fl, by_ in prof:
        d = by.setdefault(ph, [0.0, 0.0, 0.0, 0])
        d[0] += kms
        d[1] += fl
        d[2] += by_
        d[3] += 1
    total_k = sum(v[0] for v in by.values()) or 1.0
    dom = max(by, key=lambda k: by[k][0]) if by else None
    roof = None
    if dom:
        kms, fl, byt, cnt = by[dom]
        try:  # measured FMA throughput (tools/ubench_fma.cu), else unit counts x clock
            alu = json.load(open(os.path.join(ROOT, "profiles", "alu_peaks.json")))
            alu_peak = 1e12 * alu["fp64_tflops" if dtype == "c128" else "fp32_tflops"]
            alu_src = "measured (profiles/alu_peaks.json)"
        except Exception:
            lanes = 64 if dtype == "c128" else 128
            alu_peak = 148 * lanes * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6  # flop/s
            alu_src = "derived: 148 SMs x lanes x 2 x sm_max_mhz"
        hbm_peak = peaks.get("hbm_gbs", 6650.0) * 1e9
        t_alu, t_hbm = fl / alu_peak, byt / hbm_peak
        if t_alu >= t_hbm:
            ach = fl / (kms / 1e3) / 1e12
            roof = {"bound": "alu", "achieved": ach, "peak": alu_peak / 1e12, "unit": "TFLOP/s",
                    "frac": ach / (alu_peak / 1e12)}
        else:
            ach = byt / (kms / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm_peak / 1e9, "unit": "GB/s",
                    "frac": ach / (hbm_peak / 1e9)}
        jitk = {"forward": "tcx_jit_fwd_*", "backward": "tcx_jit_bwd_*", "lambda": "tcx_jit_lam_*",
                "fused": "tcx_jit_mega_*", "fused_last": "tcx_jit_mega_* (last pass)"}
        kname = {"cluster": "tcx_jit_cluster_* (cluster-resident megakernel, whole program)",
                 "dense": "dense_fwd_kernel / dense_fwd_tc_kernel (dense k-qubit blocks)",
                 "dense_backward": "dense_bwd_kernel (dense k-qubit blocks, adjoint)"}.get(
                     dom, (f"{jitk.get(dom, dom)} (per-circuit JIT window passes, {dom})"
                           if info.get("jit") else f"pass_kernel ({dom} passes)"))
        roof.update({"kernel": kname, "launches": cnt,
                     "share_of_step": kms / total_k,
                     "peak_source": alu_src if roof["bound"] == "alu" else peak_src + " (MEASURED_PEAKS.json hbm_gbs)",
                     "hbm_achieved_gbs": byt / (kms / 1e3) / 1e9,
                     "traffic": load_traffic(name, dom),
                     "algorithmic_bytes_per_launch": byt / cnt})
    kernel_split = {k: {"ms": v[0] / prof_steps, "launches_per_step": v[3] / prof_steps,
                        "tflops": v[1] / max(v[0], 1e-9) / 1e9, "gbs": v[2] / max(v[0], 1e-9) / 1e6}
                    for k, v in by.items()}
    if roof is not None and mode == "grad" and roof["bound"] == "alu":
        roof["survey_model"] = survey_flop_model(circ, H, B, ms / args.steps, alu_peak)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(circ, H, theta, mode, name, args.cpu_rows)

    launches = C.launch_count(P, B, mode == "grad") * args.steps
    line = {
        "metric": ("batched <H>+grad circuits/s (%s)" if mode == "grad" else
                   "batched <H> circuits/s (%s, forward only)") % name,
        "value": value, "unit": "circuits/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c64" if dtype == "c64" else "c128",
        "data": "synthetic",
        "config": {"workload": name, "global_batch": B * world, "batch_per_gpu": B,
                   "seq_len": None, "parallelism": f"theta-batch dp{world}",
                   "n_qubits": circ.n, "n_params": circ.n_params, "n_gates": len(circ.gates),
                   "pauli_terms": int(len(H.weights)),
                   "l2": "inputs larger than L2 (psi+lambda %.1f GiB per GPU)" % (
                       2 * B * (2 ** circ.n) * (8 if dtype == "c64" else 16) / 2 ** 30),
                   "plan": {k: info[k] for k in ("tile_bits", "reg_bits", "coalesce_bits", "fwd_passes",
                                                 "lambda_passes", "bwd_passes", "stages",
                                                 "n_ops", "jit", "dense_k", "dense_blocks")},
                   "jit_compile_s": round(t_jit, 2), "mode": mode,
                   "max_ops_per_pass": args.max_ops_per_pass, "dense_k": args.dense_k,
                   "l2_rows": args.l2_rows, "cluster_bits": args.cluster_bits,
                   "launch": graph_note + ("; per-kernel times from one extra eager profiled step"
                                           if used_graph else
                                           "; per-kernel CUDA events inside the timed region")},
        "roofline": roof,
        "kernels": kernel_split,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "circuits/s",
                "h2d_bytes_per_step": int(B * circ.n_params * 8),
                "d2h_bytes_per_step": int(B * 8 + (B * circ.n_params * 8 if mode == "grad" else 0))},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def run_sharded(args, world, rank, local, dev):
    """configs[4]: one complex64 state sharded over G ranks on its top log2 G qubits, TFIM
    <H> + adjoint grad through tcx_grad_sharded (the library runs every pass, the exchanges
    and the final sum).  N > 1: 33 + log2 N qubits (weak scaling, 2^33 amplitudes per GPU),
    library-owned NCCL communicator.  --virtual-ranks G on one GPU: the same program with G
    in-process ranks at 33 qubits in total (compare with the N = 1 line)."""
    import torch
    import torch.distributed as dist
    from paper_2205_10091_b200 import tcx
    from paper_2205_10091_b200.shard import ShardedState, exchange_counts
    G = world if world > 1 else args.virtual_ranks
    g = G.bit_length() - 1
    assert 1 << g == G, "G must be a power of two"
    n = (args.batch_qubits + g) if args.batch_qubits else (33 + g if world > 1 else 33)
    name, circ, H, theta, dtype = W.config(4, n=n)
    comm = tcx.Comm.nccl() if world > 1 else tcx.Comm.virtual(G)
    S = ShardedState(circ, H, dtype, g, comm=comm, jit=bool(args.jit), device=dev)
    t0 = time.perf_counter()
    S.C.compile(S.Pl, B=1, kind="grad")
    t_jit = time.perf_counter() - t0
    th = torch.as_tensor(theta).to(dev)
    for _ in range(args.warmup):
        S.run(th)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tcx.profile_enable(True)
    e0.record(stream)
    for _ in range(args.steps):
        E, Gr = S.run(th)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    tcx.profile_enable(False)
    prof = tcx.profile_read()
    clk = clocks.stop()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    by = {}
    for ph, idx, kms, fl, byt in prof:
        d = by.setdefault(ph, [0.0, 0.0, 0.0, 0])
        d[0] += kms
        d[1] += fl
        d[2] += byt
        d[3] += 1
    kernel_split = {k: {"ms": v[0] / args.steps, "launches_per_step": v[3] / args.steps,
                        "tflops": v[1] / max(v[0], 1e-9) / 1e9, "gbs": v[2] / max(v[0], 1e-9) / 1e6}
                    for k, v in by.items()}
    xms = by.get("exchange", [0.0])[0] / args.steps
    # e2e: theta from pinned host memory in, E / grad back, every step
    th_h = torch.as_tensor(theta).pin_memory()
    torch.cuda.synchronize(dev)
    t1 = time.perf_counter()
    for _ in range(args.steps):
        E, Gr = S.run(th_h.to(dev, non_blocking=True))
        E.cpu(), Gr.cpu()
    e2e_s = torch.tensor([time.perf_counter() - t1], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    info = S.C.info(S.Pl)
    nx1, nx3 = exchange_counts(S.C, S.Pl)
    line = {
        "metric": "sharded single-state <H>+grad circuits/s (%s)" % name,
        "value": args.steps / (ms / 1e3), "unit": "circuits/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic",
        "config": {"workload": name, "n_qubits": n, "global_bits": g, "ranks": G,
                   "virtual_ranks": world == 1,
                   "comm": "NCCL (library-owned communicator)" if world > 1 else
                           "virtual ranks (in-place swap kernels, one GPU)",
                   "plan": {k: info[k] for k in ("fwd_passes", "segments", "lambda_passes", "jit",
                                                 "exchange_overlaps")},
                   "exchange_overlap": "off (TCX_XCHG_NO_OVERLAP)" if os.environ.get("TCX_XCHG_NO_OVERLAP")
                                       else "next pass runs by chunks as they land",
                   "exchanges_per_step": {"psi": nx1, "psi_and_lambda": nx3},
                   "jit_compile_s": round(t_jit, 2),
                   "l2": "inputs larger than L2 (2^%d amplitudes per rank)" % (n - g)},
        "kernels": kernel_split,
        "exchange_ms_per_step": xms,
        "exchange_share": xms / (ms / args.steps),
        "e2e": {"value": args.steps / float(e2e_s.item()), "unit": "circuits/s",
                "h2d_bytes_per_step": int(theta.size * 8), "d2h_bytes_per_step": int(8 + theta.size * 8)},
        "gpu_launches": len(prof) // max(args.steps, 1) * args.steps,
        "clocks": clk, "cpu_baseline": None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    S.release()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def load_traffic(workload, phase):
    """DRAM bytes per launch of the dominant kernel class from a committed ncu capture
    (profiles/traffic.json via tools/summarize_profile.py), else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(workload, {}).get(phase)
    except Exception:
        return None


if __name__ == "__main__":
    sys.exit(main())
