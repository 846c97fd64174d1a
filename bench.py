"""bench.py -- whole-FMM throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--precision fp32|fp32acc|fp64]

One step = one full FMM over the configuration's synthetic cloud: tree build
(keys, sort, carve, geometry) + upward + dual traversal (lists, M2L, P2P) +
downward -- the reference's ``EvalReport.total_time`` phases
(src/traversal.py:104-106; tree build included per SPEC.md:161).

* ``value``  particles/s with the input cloud already resident in HBM
             (FP32 device tensors), timed with CUDA events per step; an L2
             flush (write of 2x L2 size) runs between steps, outside the
             event bracket.
* ``e2e``    the same metric through the public API with HOST buffers:
             ParticleSet(numpy) -> build_tree -> evaluate_on_tree ->
             results_in_input_order(), H2D/D2H inside the timed region.
* ``roofline`` of the dominant kernel (P2P): 20 flops/pair (the reference's
             cost model, src/_taylor.py:314) x p2p_pairs / P2P kernel time
             (events on the launching stream), against the FP32 FMA peak
             measured live by an FFMA probe kernel at the running clock.
* ``cpu_baseline`` the C oracle restating the reference (oracle/fmm_oracle.c)
             on this host's cores, bounded sample.

Multi-GPU (torchrun, one rank per GPU): the target leaves are split into
contiguous Morton ranges; every rank builds the (identical) tree, computes
its own rows and the max over ranks is reported (scaling "strong").
``--impl reference`` runs the reference's algorithm on the host CPU (the C
oracle, all threads) on rank 0 only.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1209_3516_b200 import workloads  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "p2p_traffic.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--n", type=int, default=0, help="override N (testing)")
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp32acc", "fp64"])
    ap.add_argument("--p", type=int, default=0, help="override the expansion order (C4 sweep)")
    ap.add_argument("--theta", type=float, default=0.0, help="override theta (C4 sweep)")
    ap.add_argument("--strategy", default="dualtree", choices=["dualtree", "treecode", "listfmm"],
                    help="evaluation strategy (the headline is the dual-tree FMM)")
    ap.add_argument("--mutual", action="store_true", help="mutual dual traversal (EvalConfig.mutual)")
    ap.add_argument("--symmetric", action="store_true",
                    help="with --mutual: symmetric near field over the unordered mutual pairs (EvalConfig.symmetric)")
    ap.add_argument("--sharded", action="store_true",
                    help="N>1: each rank gets only its block of the input and keeps only its own bodies plus "
                         "the near-field halo (paper_1209_3516_b200.sharded) instead of the replicated cloud")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: the configuration's N per GPU (N x WORLD_SIZE bodies in all; BASELINE "
                         "configs[4]: --config C5 --n 4194304 --weak), reported as \"scaling\": \"weak\"")
    ap.add_argument("--task-grain", type=int, default=5000, help="EvalConfig.task_grain (mutual partition)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-accuracy", action="store_true", help="skip the 1000-sample direct-sum check")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="target CPU work for the baseline sample")
    return ap.parse_args()


def workload(args):
    gen, n, solver = workloads.CONFIGS[args.config]
    n = args.n or n
    if getattr(args, "weak", False):
        n *= int(os.environ.get("WORLD_SIZE", "1"))
    pos, q = gen(n, 0)
    solver = dict(solver)
    if args.p:
        solver["p"] = args.p
    if args.theta:
        solver["theta"] = args.theta
    return pos, q, n, solver


def config_block(args, n, solver, extra=None):
    d = {"workload": f"{args.config}: Laplace FMM N={n}", "n": n, "p": solver["p"], "theta": solver["theta"],
         "ncrit": solver["ncrit"], "mac": "fmm", "strategy": getattr(args, "strategy", "dualtree"),
         "distribution": {"C1": "uniform f64", "C2": "uniform f32, q~U[0,1)", "C3": "Plummer a=1 rcut=10a",
                          "C4": "uniform f32, q~U[-1,1)", "C5": "uniform f32, q~U[0,1)"}[args.config],
         "l2": "flushed between timed steps (2x L2 write)"}
    if getattr(args, "mutual", False):
        d.update(mutual=True, task_grain=args.task_grain, symmetric=bool(getattr(args, "symmetric", False)))
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            q = os.environ.get("FMM_BENCH_CLOCK_Q", self.Q)
            if q == "none":
                raise RuntimeError("sampler disabled")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms",
                                          os.environ.get("FMM_BENCH_CLOCK_MS", "50")],
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
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline: the C oracle on host cores
# ---------------------------------------------------------------------------
def cpu_run(pos, q, solver, seconds_target, threads=0):
    """Bounded sample of the reference algorithm on the host; returns
    (particles_per_s, details).  Build, upward and list collection run in
    full; M2L/P2P/L2P run for a Morton prefix of target leaves (tfrac) and
    are extrapolated linearly to all targets."""
    from oracle import oracle as orc
    n = pos.shape[0]
    nthr = threads or orc.max_threads()
    probe = orc.fmm(pos, q, solver["ncrit"], solver["p"], solver["theta"], threads=nthr, tfrac=0.002)
    t = probe["times"]
    frac_done = probe["bodies_done"] / n
    per_full = (t["m2l"] + t["p2p"] + t["downward"]) / max(frac_done, 1e-9)
    fixed = t["build"] + t["upward"] + t["lists"]
    tfrac = min(1.0, max(0.002, (seconds_target - fixed) / max(per_full, 1e-9)))
    r = orc.fmm(pos, q, solver["ncrit"], solver["p"], solver["theta"], threads=nthr, tfrac=tfrac)
    t = r["times"]
    frac_done = r["bodies_done"] / n
    total = t["build"] + t["upward"] + t["lists"] + (t["m2l"] + t["p2p"] + t["downward"]) / frac_done
    return n / total, dict(tfrac=tfrac, bodies_done=r["bodies_done"], times=t, threads=nthr,
                          est_total_s=total, p2p_pairs_sampled=r["p2p_pairs"])


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    pos, q, n, solver = workload(args)
    vals = []
    # bounded: the whole --steps K --warmup W run stays around three minutes
    per_step = max(2.0, min(args.cpu_seconds, 180.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_run(pos, q, solver, per_step)
    details = None
    for _ in range(args.steps):
        v, details = cpu_run(pos, q, solver, per_step)
        vals.append(v)
    value = float(np.median(vals))
    line = {
        "impl": "reference", "metric": "FMM particles/s (Laplace, P=%d)" % solver["p"], "value": value,
        "unit": "particles/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * n / value, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_block(args, n, solver),
        "cpu_baseline": {"value": value, "unit": "particles/s", "cores": details["threads"], "kind": "port",
                         "sample": f"C oracle (restated reference, OpenMP {details['threads']} threads, {cpu_model()}): "
                                   f"full build/upward/lists + M2L/P2P/L2P on a Morton prefix of "
                                   f"{details['bodies_done']} of {n} targets, extrapolated"},
        "e2e": {"value": value, "unit": "particles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def fp32_peak(torch, lib_call, stream):
    """Measured FP32 FMA peak (TFLOP/s) of this GPU at the running clock:
    the better of the FFMA and FFMA2 probes."""
    import ctypes as C
    from paper_1209_3516_b200 import _lib
    sink = torch.zeros(148 * 64, dtype=torch.float32, device="cuda")
    best = {}
    names = {0: "ffma_imm", 1: "ffma2_imm", 2: "ffma_reg", 3: "ffma2_reg", 4: "fmul_fadd_reg"}
    for packed in (0, 1, 2, 3, 4):
        flops = C.c_double(0)
        for _ in range(2):
            lib_call("fmm_ffma_probe", packed, 148 * 16, 4096, _lib.ptr(sink), C.byref(flops), stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            lib_call("fmm_ffma_probe", packed, 148 * 16, 4096, _lib.ptr(sink), C.byref(flops), stream)
        e1.record()
        e1.synchronize()
        best[names[packed]] = 5 * flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12
    return max(best["ffma_imm"], best["ffma2_imm"]), best


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1209_3516_b200 as fb
    from paper_1209_3516_b200 import _lib
    from paper_1209_3516_b200 import distributed as fdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FMM_BENCH_BACKEND / FMM_BENCH_SAME_DEVICE exist for testing the
    # multi-rank code path on a one-GPU box (gloo, every rank on cuda:0);
    # the driver's runs use NCCL with one GPU per rank
    if os.environ.get("FMM_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("FMM_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    pos, q, n, solver = workload(args)
    cfg = fb.EvalConfig(strategy=args.strategy, mac=fb.MacConfig("fmm", solver["theta"]), p=solver["p"],
                        precision=args.precision, mutual=args.mutual, task_grain=args.task_grain,
                        symmetric=bool(args.mutual and args.symmetric))
    dev = torch.device("cuda", local)
    dt = torch.float32 if pos.dtype == np.float32 else torch.float64
    dpos = torch.as_tensor(pos, device=dev).to(dt)
    ps_dev = fb.ParticleSet(dpos[:, 0].contiguous(), dpos[:, 1].contiguous(), dpos[:, 2].contiguous(),
                            torch.as_tensor(q, device=dev).to(dt))
    flush = torch.empty(2 * 126 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    sharded = args.sharded and world > 1
    if sharded:
        from paper_1209_3516_b200 import sharded as fsh
        blk = slice(rank * n // world, (rank + 1) * n // world)  # this rank's block of the input
        shard_dev = [dpos[blk, 0].contiguous(), dpos[blk, 1].contiguous(), dpos[blk, 2].contiguous(),
                     torch.as_tensor(q[blk], device=dev).to(dt)]

    def step():
        if sharded:
            tree = fsh.build_tree_sharded(*shard_dev, solver["ncrit"], rank, world, device=dev)
            rep, _ = fsh.evaluate_sharded(tree, cfg, results="local")
            return tree, rep
        tree = fb.build_tree(ps_dev, ncrit=solver["ncrit"])
        if world > 1:
            rep = fdist.evaluate_partitioned(tree, cfg, rank, world, results="root")
        else:
            rep = fb.evaluate_on_tree(tree, cfg)
        return tree, rep

    clocks = Clocks(local)
    # the interpreter's cyclic GC stays out of the timed steps (as in
    # timeit): a full collection over torch's object graph is a ~15 ms host
    # pause that leaves the GPU idle (seen as one slow step in ten)
    gc.collect()
    gc.freeze()
    gc.disable()
    clocks.start()  # sampled through warm-up and the timed region (both under load)
    # at least W warm-up steps, and at least 5: the caching allocator settles
    # its block layout over the first four evaluations (two trees alive while
    # a step builds the next); a fifth keeps its last cudaMalloc (C2 32 MB,
    # C3 128 MB) out of the first timed step (tools/alloc_probe.py)
    warm = max(5, args.warmup)
    for _ in range(warm):
        tree, rep = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times, p2p_times, reps = [], [], []
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        tree, rep = step()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1) * 1e-3)
        p2p_times.append(rep.stats.times.get("p2p", float("nan")))
        reps.append(rep)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total = max_over_ranks(float(np.sum(times)))
    ms = 1e3 * total / args.steps
    value = n * args.steps / total
    rep = reps[-1]

    # e2e through the public API with host buffers (every rank holds the
    # whole host cloud, as the replicated build needs; rank 0 reads back the
    # gathered results; the time is the max over ranks)
    e2e = None
    if not args.no_e2e:
        # host arrays in the configuration's precision (float32 for C2-C5):
        # ParticleSet keeps them as given and the device upcasts them
        # ... in page-locked memory (the bench contract's "from pinned host
        # memory"; FMM_BENCH_PAGEABLE=1 keeps pageable arrays, which build_tree
        # stages through its own pinned buffers)
        def host(a):
            a = np.ascontiguousarray(a)
            if os.environ.get("FMM_BENCH_PAGEABLE") == "1":
                return a
            h = torch.empty(a.shape, dtype=torch.from_numpy(a).dtype, pin_memory=True).numpy()
            h[...] = a
            return h

        hx, hy, hz = (host(pos[:, k]) for k in range(3))
        hq = host(q)
        h2d = sum(a.nbytes for a in (hx, hy, hz, hq))

        def e2e_step():
            if sharded:  # the rank's block in, its block's (phi, f) back
                b = slice(rank * n // world, (rank + 1) * n // world)
                tr = fsh.build_tree_sharded(hx[b], hy[b], hz[b], hq[b], solver["ncrit"], rank, world, device=dev)
                _, res = fsh.evaluate_sharded(tr, cfg, results="input")
                return [r.cpu().numpy() for r in res]
            ps = fb.ParticleSet(hx, hy, hz, hq)
            tr = fb.build_tree(ps, ncrit=solver["ncrit"])
            if world > 1:
                fdist.evaluate_partitioned(tr, cfg, rank, world, results="root")
                return tr.results_in_input_order() if rank == 0 else None
            fb.evaluate_on_tree(tr, cfg)
            return tr.results_in_input_order()

        for _ in range(4):
            e2e_step()
        torch.cuda.synchronize()
        et = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            res = e2e_step()
            et.append(max_over_ranks(time.perf_counter() - t0))
        e2e = {"value": n / float(np.median(et)), "unit": "particles/s",
               "h2d_bytes_per_step": h2d if sharded else h2d * world, "d2h_bytes_per_step": 4 * 8 * n,
               "note": "ParticleSet(host numpy in pinned memory) -> build_tree -> evaluate_on_tree (evaluate_partitioned over the "
                       "ranks, results gathered to rank 0) -> results_in_input_order() (phi, f back in input "
                       "order as float64); wall clock per "
                       "step, median of the max over ranks"}
        del res

    gc.enable()
    # accuracy of the last timed step: relative L2 error against direct
    # summation on the reference's 1000-body sample (tree order, seed 0)
    acc = None
    if rank == 0 and not args.no_accuracy and not sharded:  # (sharded: rank 0 holds only its rows)
        from paper_1209_3516_b200.tuner import potential_sample, sampled_force_error, sampled_potential_error
        idx, fref, pref = potential_sample(tree, 1000, 0)
        acc = {"force_err": sampled_force_error(tree, idx, fref), "pot_err": sampled_potential_error(tree, idx, pref),
               "sample": int(idx.size), "reference": "direct O(N*S) sums on the GPU, FP64 (src/tuner.py:30-55)"}

    peak, peaks = fp32_peak(torch, _lib.call, sh)
    p2p_s = float(np.median(p2p_times))
    achieved = 20.0 * rep.stats.p2p_pairs / p2p_s / 1e12
    # target slots the near field computes per real target: a leaf of c
    # bodies runs as blocks of 8 with a last block of 4 or 8, i.e. 4*ceil(c/4)
    # slots (DESIGN.md (f) 1); `frac` counts real pairs only
    leaf_cnt = (tree.d_end - tree.d_start)[tree.d_leaf.bool()].long()
    slot_ratio = float((((leaf_cnt + 3) // 4) * 4).sum().item()) / max(float(leaf_cnt.sum().item()), 1.0)
    traffic = None
    if os.path.exists(TRAFFIC_PATH):
        try:
            traffic = json.load(open(TRAFFIC_PATH)).get(args.config, {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1 and args.strategy == "dualtree" and not args.mutual:
        v, d = cpu_run(pos, q, solver, args.cpu_seconds)
        v1, d1 = cpu_run(pos, q, solver, args.cpu_seconds / 2, threads=1)
        cpu = {"value": v, "unit": "particles/s", "cores": d["threads"], "kind": "port",
               "sample": f"C oracle (restated reference, {d['threads']} threads, {cpu_model()}): full "
                         f"build/upward/lists, M2L/P2P/L2P on {d['bodies_done']}/{n} targets (Morton prefix), "
                         f"extrapolated",
               "single_thread": {"value": v1, "unit": "particles/s", "cores": 1,
                                 "sample": f"same, 1 thread, {d1['bodies_done']}/{n} targets, extrapolated"}}
    kernel_ms = {k: 1e3 * v for k, v in rep.stats.times.items()}
    line = {
        "metric": "FMM particles/s (Laplace, P=%d)" % solver["p"], "value": value, "unit": "particles/s",
        "n_gpus": world, "steps": args.steps, "warmup": warm, "ms_per_step": ms,
        "step_ms": {"min": 1e3 * float(np.min(times)), "median": 1e3 * float(np.median(times)),
                    "max": 1e3 * float(np.max(times)), "all": [round(1e3 * t, 3) for t in times]},
        "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
        "dtype": {"fp32": "f32 P2P / f64 tree+far field", "fp32acc": "f32 P2P terms, f64 sums / f64 tree+far field",
                  "fp64": "f64"}[args.precision],
        "data": "synthetic", "config": config_block(args, n, solver, {"precision": args.precision,
                                                                      "parallelism": f"morton-partition x{world}"
                                                                      + (" sharded+halo" if sharded else "")}),
        "p2p_ginteractions_per_s": rep.stats.p2p_pairs / p2p_s / 1e9,
        "p2p_pairs": rep.stats.p2p_pairs, "m2l_calls": rep.stats.m2l_calls, "m2p_calls": rep.stats.m2p_calls,
        "phase_ms": {"build": 1e3 * rep.build_time, "upward": 1e3 * rep.upward_time,
                     "traversal": 1e3 * rep.traversal_time, "downward": 1e3 * rep.downward_time},
        # EvalReport.total_time (the reference's N / total_time metric) per timed step, against the
        # event-timed step above; the phases are the critical-path split of the overlapped evaluation
        "report_total_ms": {"median": 1e3 * float(np.median([r.total_time for r in reps])),
                            "vs_ms_per_step": float(np.median([r.total_time for r in reps])) / (ms * 1e-3)},
        "stream_spans_ms": {k: 1e3 * v for k, v in rep.spans.items()},
        "near_field_precision": rep.near_field,
        "kernel_ms": kernel_ms,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "target_slots_per_target": slot_ratio, "frac_with_padded_slots": achieved * slot_ratio / peak,
                     "peak_source": "FFMA/FFMA2 probe measured live in this run (%s); MEASURED_PEAKS.json has "
                                    "no FP32 figure" % ", ".join(f"{k} {v:.1f}" for k, v in peaks.items()),
                     "kernel": "p2p_f32_kernel", "flop_model": "20 flops/pair (src/_taylor.py:314)"},
        "accuracy": acc, "e2e": e2e, "cpu_baseline": cpu, "clocks": clk,
        "gpu_launches": launches,
        "gpu_launches_per_step": launches / args.steps,
    }
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
