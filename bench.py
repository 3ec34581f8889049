#!/usr/bin/env python
"""Benchmark of the hot path: count the models of a Boolean program over all
2^n valuations of the free generators (arXiv 1310.6978 §2.3, Prop 2.2).

Default workload (the config BASELINE.json's metric is quoted on: register
mode count at 1/2/4/8 GPUs against the int-ALU roofline) is config C5: a
random 1000-gate Boolean DAG over n = 42 variables, 2^42 valuations per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5|c4|c3_posets|c2|c2_n32|...]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)
    python bench.py --impl reference ...                   (the CPU oracle arm)

Headline (`value`): the paper's brute-force block evaluation (PAPER.md:356-372,
955) -- ONE register-mode kernel (presets.exhaustive(config): generators synthesised
in registers, 2^slot_bits slot cofactors folded into a straight-line LOP3/IMAD body,
searched variable roles, fused popcount + reduction) evaluates every word of
every valuation of the rank's cofactor range [r 2^(n-p), (r+1) 2^(n-p)) inside
the timed region; then ONE 8-byte NCCL all-reduce (P > 1).  Nothing is decided
at preparation time.  Preparation (role search + NVRTC, rank 0 first so the
other ranks load its cubin from the JIT cache) is outside the timed region and
reported as prep_s, as in any JIT-compiled benchmark.

`e2e`: a COLD call through the public API, every step: bfa_compile of the
text -> bfa_count_range with the plan of least preparation + one count
(presets.cold: role search + PTX compile with the persistent JIT cache
disabled, module load, launch) -> the count read on the host (and, P > 1,
all-reduced); wall clock, max over ranks.

`replay` (N = 1, C5/C4): the decomposed plan (presets.DECOMPOSED: Shannon
leaves of the Reduction run as work-queue kernels).  Leaves the Reduction
proves 0 are decided during its preparation, so its step time is a replay of
a prepared plan; reported with its cold preparation time and the valuations
it decided, never as the headline.

Timing: W untimed warm-up steps; L2 flushed (256 MiB write) between timed
steps; CUDA events on the launching stream; barrier + synchronize on both
sides; max over ranks.  Prints one JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

SMS = 148


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bfa", choices=["bfa", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the replay and the extra config lines")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo + --share-device: functional multi-rank runs on one GPU)")
    ap.add_argument("--share-device", action="store_true",
                    help="every rank on cuda:0 (functional test of the N > 1 path on a one-GPU box; not a "
                         "scaling measurement)")
    ap.add_argument("--options", default=None,
                    help="JSON dict of program options applied on top of the preset (profiling variants)")
    return ap.parse_args()


MATERIALISED = {"c2": ("c2", 0), "c2_fused": ("c2", 1), "c2_n32": ("c2_n32", 0), "c2_n32_fused": ("c2_n32", 1)}

CONFIG_DESC = {
    "c1": "labeled partial orders on 3 points, n=9 (BASELINE configs[0])",
    "c2": "random 3-CNF, 2000 clauses over n=28, materialised vector algebra (HBM) + popcount (BASELINE configs[1])",
    "c2_fused": "random 3-CNF, 2000 clauses over n=28, materialised table S, fused 128-bit-load kernel + popcount",
    "c2_n32": "random 3-CNF, 2000 clauses over n=32 (512 MiB vectors >> L2), materialised vector algebra + popcount",
    "c2_n32_fused": "random 3-CNF, 2000 clauses over n=32, materialised table S, fused kernel + popcount",
    "c5": "random 1000-gate Boolean DAG over n=42 vars, count mode (BASELINE configs[4])",
    "c4": "labeled partial orders on 6 points, n=36, count mode (BASELINE configs[3])",
    "c3_posets": "labeled partial orders on 5 points, n=25, count mode (BASELINE configs[2])",
    "c3_equiv": "equivalence relations on 5 points, n=25, count mode (BASELINE configs[2])",
    "paper_2p17": "the paper's timed experiment shape: a 30-variable term with 2^17 tree nodes, all 2^30 valuations "
                  "(PAPER.md:374-380; ~1 s on the paper's 2-GPU rig), segmented execution",
}


def config_block(name, n, world):
    """Workload identity only (identical in both arms)."""
    return {"workload": f"{name}: {CONFIG_DESC.get(name, name)}", "n": n, "valuations_per_step": 1 << n,
            "seed": W.SEED, "parallelism": f"cofactor x{world} (top log2(P) variable ids, contiguous ranges)",
            "l2": "count mode reads no HBM inputs (generators synthesised in registers); "
                  "L2 flushed with a 256 MiB write before every timed step anyway"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [r for r in self.rows if len(r) >= 8]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[4 + k] == "Active"})
        pw = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------- oracle (CPU) leg
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def _subcube(n, k, i, count):
    """Start of the i-th of `count` spread-out aligned 2^k sub-cubes of [0, 2^n)."""
    if k >= n:
        return 0
    slots = 1 << (n - k)
    return ((i * slots) // count + (slots // (2 * count))) % slots << k


def oracle_rate(text, n, seconds, threads=None, cubes=4):
    """Time the CPU oracle, as it stands, on a bounded sample of the workload:
    `cubes` spread-out aligned sub-cubes, sized together for ~`seconds` of
    CPU work.  Returns (valuations/s, threads, description)."""
    import oracle
    threads = threads or oracle.default_threads()
    k = min(12, n)
    while True:                                   # size probe
        t0 = time.perf_counter()
        oracle.count(text, n, 0, 1 << k, threads=threads)
        dt = time.perf_counter() - t0
        if dt > 0.3 or k >= n:
            break
        k = min(k + 2, n)
    rate = (1 << k) / max(dt, 1e-9)
    k2 = min(n, max(k, int(rate * seconds / cubes).bit_length() - 1))
    m = 1 if k2 >= n else cubes
    total, spent, starts = 0, 0.0, []
    for i in range(m):
        lo = _subcube(n, k2, i, m)
        starts.append(lo)
        t0 = time.perf_counter()
        oracle.count(text, n, lo, lo + (1 << k2), threads=threads)
        spent += time.perf_counter() - t0
        total += 1 << k2
    desc = (f"{m} sub-cubes of 2^{k2} valuations at mu = {starts[:4]}{'...' if m > 4 else ''} "
            f"({total} valuations, {spent:.1f} s)")
    if m == 1 and k2 >= n:
        desc = f"sub-cube of 2^{k2} valuations [0, {1 << k2}), {spent:.1f} s (the whole cube)"
    return total / spent, threads, desc


def cpu_baseline_block(text, n, seconds):
    """The oracle on the host: all-cores rate on >= 4 sub-cubes, a 1-thread
    rate, the CPU model, and the extrapolated full-run time."""
    import oracle
    allc = oracle.default_threads()
    v, cores, sample = oracle_rate(text, n, seconds * 0.75, threads=allc)
    v1, _, sample1 = oracle_rate(text, n, seconds * 0.25, threads=1, cubes=1)
    return {"value": v, "unit": "valuations/s", "cores": cores, "kind": "oracle", "sample": sample,
            "one_thread": {"value": v1, "sample": sample1}, "cpu_model": cpu_model(),
            "extrapolated_full_run_s": (1 << n) / v}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    text, n, _ = W.config(args.config)
    steps = []
    for i in range(args.warmup + args.steps):
        v, cores, sample = oracle_rate(text, n, args.cpu_seconds / 3)
        if i >= args.warmup:
            steps.append(v)
    value = statistics.median(steps)
    line = {"impl": "reference", "metric": "valuations/s", "value": value, "unit": "valuations/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": (1 << n) / value * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bool (C int per valuation)", "data": "synthetic",
            "config": config_block(args.config, n, 1),
            "cpu_baseline": {"value": value, "unit": "valuations/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "valuations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def ncu_alu_for(cfg):
    """ALU-pipe utilisation of the kernel from the committed ncu --set full
    capture (profiles/traffic.json): SURVEY 8(d)'s executed-instruction
    fraction (every ALU-pipe instruction, loop and popcount included), next
    to the cover-cell fraction measured live."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            e = json.load(f)[cfg]
        return dict(e["ncu_alu_pipe"], source=e["source"])
    except (OSError, KeyError, ValueError):
        return None


def traffic_for(cfg):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[cfg]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


# ---------------------------------------------------------------- GPU helpers
def measure_int_peaks(bfa, torch, dev):
    """Measured integer issue rates (ops/s): LOP3 only (ALU pipe), IMAD only
    (FMA pipe), and LOP3+IMAD 1:1 (both pipes, bounded by issue)."""
    sink = torch.zeros(4096, dtype=torch.int32, device=dev)
    blocks, threads, iters = SMS * 8, 256, 2000
    out = {}
    for op, name in ((0, "lop3"), (1, "imad"), (2, "lop3_imad_1to1")):
        bfa.peak_int(op, blocks, threads, 10, sink)
        torch.cuda.synchronize()
        best = 0.0
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            bfa.peak_int(op, blocks, threads, iters, sink)
            e.record()
            torch.cuda.synchronize()
            best = max(best, blocks * threads * iters * 256 / (s.elapsed_time(e) / 1e3))
        out[name] = best
    return out


def int_roofline(launch, words, seconds, peaks, cfg):
    """Roofline of a register-mode count: algorithmic work per 32-bit word =
    the executed cells of the slot-cofactored, hoisted cover:
    A LOP3 cells on the ALU pipe and F IMAD cells (+ IMAD operand registers)
    on the FMA pipe.  The bound for this mix is the binding one of
    R_lop3 / A, R_imad / F and R_issue / (A + F) words/s (measured rates)."""
    A = launch["cells_lop3"] / words
    F = launch["cells_imad"] / words
    wps = words / seconds
    terms = {"alu_pipe (LOP3)": peaks["lop3"] / A if A else float("inf"),
             "fma_pipe (IMAD)": peaks["imad"] / F if F else float("inf"),
             "issue (1 warp-inst/clk/SMSP)": peaks["lop3_imad_1to1"] / (A + F)}
    binding = min(terms, key=terms.get)
    bound = terms[binding]
    return {"bound": "alu", "achieved": (A + F) * wps, "peak": (A + F) * bound, "unit": "int ops/s",
            "frac": wps / bound, "traffic": traffic_for(cfg),
            "per_unit": f"{A + F:.2f} integer cells per 32-bit word (32 valuations): {A:.2f} LOP3 (ALU pipe) + "
                        f"{F:.2f} IMAD (FMA pipe) of the slot-cofactored, hoisted cover",
            "units_per_launch": words, "binding": binding,
            "peak_source": "measured bfa_peak_int rates (LOP3 ALU pipe, IMAD FMA pipe, 1:1 mix issue-bound); "
                           "peak = the binding pipe for this kernel's LOP3:IMAD mix",
            "peak_measured": peaks,
            "ncu_alu_pipe": ncu_alu_for(cfg),
            "alu_pipe": {"lop3_per_s": A * wps, "frac": A * wps / peaks["lop3"]},
            "fma_pipe": {"imad_per_s": F * wps, "frac": F * wps / peaks["imad"]}}


class Timer:
    """CUDA events on one stream around each of K steps; L2 flushed between."""

    def __init__(self, torch, stream, dev):
        self.torch, self.stream = torch, stream
        self.flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def run(self, fn, steps):
        torch = self.torch
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            self.flush.fill_(i & 0xFF)
            ev[i][0].record(self.stream)
            fn()
            ev[i][1].record(self.stream)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) / 1e3 for s, e in ev]


def run_bfa(args):
    import torch
    import torch.distributed as dist

    import paper_1310_6978_b200 as bfa
    from paper_1310_6978_b200 import presets
    from paper_1310_6978_b200.dist import prepare_sharded, rank_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    gpu = 0 if args.share_device else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")

    text, n, expect = W.config(args.config)
    extra_opts = json.loads(args.options) if args.options else {}
    preset = presets.exhaustive(args.config)
    prog = presets.apply(bfa.Program(text), preset, **extra_opts)
    info = prog.info
    lo, hi = rank_range(n, rank, world)
    stream = torch.cuda.current_stream()
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)

    def step():
        prog.count_range(n, lo, hi, out=cnt, stream=stream)
        if world > 1:
            dist.all_reduce(cnt)

    # ---- preparation (role search + NVRTC + module load), untimed.  Rank 0
    # compiles first and writes the persistent JIT cache; the other ranks then
    # load its role search and cubin instead of re-deriving them.
    t_prep = time.perf_counter()
    if world > 1:
        prepare_sharded(prog, n)            # rank 0 compiles, the others load its results
    prog.count_range(n, lo, hi, out=cnt, stream=stream)
    torch.cuda.synchronize()
    prep_s = time.perf_counter() - t_prep
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launch = bfa.last_launch()

    timer = Timer(torch, stream, dev)
    clocks = ClockSampler(gpu)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = bfa.last_launch().get("launch_counter", 0)
    clocks.start()
    time.sleep(0.3)
    step_s = timer.run(step, args.steps)
    launches_timed = bfa.last_launch().get("launch_counter", 0) - launches0
    clk = clocks.stop()
    # kernel-only time of this rank (the count without the all-reduce)
    kern_s = timer.run(lambda: prog.count_range(n, lo, hi, out=cnt, stream=stream), min(args.steps, 5))
    if world > 1:
        step()
        dist.barrier()
    t_total, t_kern = sum(step_s), statistics.median(kern_s)
    if world > 1:
        tt = torch.tensor([t_total, t_kern], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total, t_kern = tt.tolist()
    final = int(cnt.item()) & ((1 << 64) - 1)
    value = (1 << n) * args.steps / t_total
    words = (hi - lo) >> 5
    peaks = measure_int_peaks(bfa, torch, dev)
    roof = int_roofline(launch, words, t_kern, peaks, args.config + "_exhaustive")

    # ---- e2e: COLD call through the public API every step (compile -> count
    # -> host), persistent JIT cache disabled, max over ranks
    e2e_steps = max(1, args.e2e_steps)
    cubin_bytes = 0
    e2e_t = []
    for _ in range(e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = presets.apply(bfa.Program(text), presets.cold(args.config), jit_cache=0, **extra_opts)
        t = q.count_range(n, lo, hi, stream=stream)
        if world > 1:
            dist.all_reduce(t)
        e2e_count = int(t.item()) & ((1 << 64) - 1)   # device -> host read (synchronises)
        e2e_t.append(time.perf_counter() - t0)
        cubin_bytes = len(q.jit_cubin(1, n)) if world == 1 else 0   # (cached: no recompile)
        assert e2e_count == final, (e2e_count, final)
        del q
    e2e_s = statistics.median(e2e_t)
    if world > 1:
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_s = te.item()
    # for comparison: one cold call with the value plan (long preparation)
    e2e_value_plan = None
    if world == 1 and not args.no_extras:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = presets.apply(bfa.Program(text), preset, jit_cache=0, **extra_opts)
        t = q.count_range(n, lo, hi, stream=stream)
        ok = (int(t.item()) & ((1 << 64) - 1)) == final
        dt = time.perf_counter() - t0
        e2e_value_plan = {"s_per_call": dt, "valuations_per_s": (1 << n) / dt, "count_equal": ok,
                          "what": "one cold call (compile -> count -> host) with the value plan instead of "
                                  "presets.cold: longer role search and compile, faster kernel"}
        del q

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    verified = {}
    if expect is not None:
        verified["closed_form"] = final == expect
        assert final == expect, (final, expect)

    extras = {}
    if world == 1 and not args.no_extras:
        extras = run_extras(args, bfa, presets, torch, stream, dev, text, n, final, verified, peaks, timer)

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline_block(text, n, args.cpu_seconds)

    line = {
        "metric": "valuations/s", "value": value, "unit": "valuations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32 (bitwise LOP3/IMAD on 32-valuation words)",
        "data": "synthetic (seeded generator, workloads/__init__.py)",
        "config": dict(config_block(args.config, n, world),
                       **({"functional_multi_rank": f"{world} ranks sharing cuda:0 over {args.backend}: checks the "
                                                    "N > 1 path, not a scaling measurement"}
                          if args.share_device and world > 1 else {})),
        "program": {"gates_G": info["gates"], "luts_L": info["luts"], "support": info["support"],
                    "options": dict(preset, **extra_opts)},
        "gate_word_ops": {
            "nominal_per_s": info["gates"] * value / 32, "lut3_level_per_s": info["luts"] * value / 32,
            "lop3_peak_per_s": peaks["lop3"],
            "note": "SURVEY 8(d): G (gates) and L (LUT3 cells of the unspecialised cover) x 32-bit words per "
                    "second. Both exceed the LOP3 peak: slot cofactoring and loop hoisting execute "
                    "roofline.per_unit cells per word instead of L, so they are nominal, not executed, rates"},
        "count": final, "count_expected": expect, "count_verified": verified,
        "decided_at_compile_time": 0,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": (1 << n) / e2e_s, "unit": "valuations/s", "h2d_bytes_per_step": cubin_bytes,
                "d2h_bytes_per_step": 8, "steps": e2e_steps, "s_per_call": e2e_s,
                "plan": dict(presets.cold(args.config), **extra_opts),
                "call": "cold: bfa_compile(text) -> bfa_count_range over this rank's range with the plan of least "
                        "preparation + one count (presets.cold: role search + PTX compile with the persistent JIT "
                        "cache off, module load, launch) -> count read on the host"
                        + (" -> all-reduce" if world > 1 else ""),
                "h2d": "the JIT'd cubin loaded into the device each call (count mode has no input tensors)",
                "value_plan": e2e_value_plan},
        "gpu_launches": launches_timed,
        "kernel_ms_per_step": t_kern * 1e3,
        "prep_s": prep_s,
        "launch": launch,
        "clocks": clk,
    }
    line.update(extras)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_extras(args, bfa, presets, torch, stream, dev, text, n, final, verified, peaks, timer):
    """Secondary measurements in the same run (N = 1): the decomposed plan as
    a labelled replay, the exhaustive line of the other count config, and
    the materialised mode of C2 (HBM)."""
    out = {}
    steps = max(3, min(args.steps, 5))
    if args.config in ("c5", "c4"):
        # complement invariant through the same exhaustive preset (P-11)
        body, outl = "\n".join(text.splitlines()[:-1]), text.splitlines()[-1]
        if args.config == "c5":
            pc = presets.apply(bfa.Program(f"{body}\n~{outl}"), presets.exhaustive(args.config))
            verified["complement_sum"] = final + pc.count(n) == 1 << n
        # the decomposed plan, cold preparation, then replays
        q = presets.apply(bfa.Program(text), presets.DECOMPOSED, jit_cache=0)
        c = torch.zeros(1, dtype=torch.int64, device=dev)
        t0 = time.perf_counter()
        q.count_range(n, 0, 1 << n, out=c, stream=stream)
        torch.cuda.synchronize()
        prep = time.perf_counter() - t0
        for _ in range(2):
            q.count_range(n, 0, 1 << n, out=c, stream=stream)
        torch.cuda.synchronize()
        ll = bfa.last_launch()
        ts = timer.run(lambda: q.count_range(n, 0, 1 << n, out=c, stream=stream), steps)
        rc = int(c.item())
        verified["decomposed_equals_exhaustive"] = rc == final
        decided = ll.get("valuations_decided", 0)
        t = statistics.median(ts)
        out["replay"] = {
            "what": "REPLAY of a prepared Shannon-decomposition plan (presets.DECOMPOSED): leaves the Reduction "
                    "proved 0 were decided during preparation; not the headline",
            "ms_per_step": t * 1e3, "valuations_per_s": (1 << n) / t,
            "executed_valuations_per_s": ((1 << n) - decided) / t, "valuations_decided_at_prep": decided,
            "prep_s_cold": prep, "first_call_valuations_per_s": (1 << n) / (prep + t), "count": rc,
            "kernels": ll.get("kernels"), "queue": ll.get("queue"), "decompose_s": ll.get("decompose_s"),
            "roofline": int_roofline(ll, 1 << (n - 5), t, peaks, args.config + "_replay")}
    if args.config == "c5":
        # the exhaustive line at n = 36 (C4)
        t4, n4, e4 = W.config("c4")
        p4 = presets.apply(bfa.Program(t4), presets.exhaustive("c4"))
        c4 = torch.zeros(1, dtype=torch.int64, device=dev)
        for _ in range(3):
            p4.count_range(n4, 0, 1 << n4, out=c4, stream=stream)
        torch.cuda.synchronize()
        l4 = bfa.last_launch()
        ts = timer.run(lambda: p4.count_range(n4, 0, 1 << n4, out=c4, stream=stream), max(args.steps, 10))
        t = statistics.median(ts)
        verified["c4_closed_form"] = int(c4.item()) == e4
        out["c4_exhaustive"] = {"valuations_per_s": (1 << n4) / t, "ms_per_step": t * 1e3, "count": int(c4.item()),
                                "roofline": int_roofline(l4, 1 << (n4 - 5), t, peaks, "c4_exhaustive")}
        out["c4_eval"] = eval_line(bfa, torch, stream, dev, p4, n4, e4, max(args.steps, 5), timer, verified)
        del p4
        for name in ("c2", "c2_fused", "c2_n32", "c2_n32_fused"):
            out[name] = materialised_line(bfa, torch, stream, name, 3, timer)
    return out


def eval_line(bfa, torch, stream, dev, prog, n, expect, steps, timer, verified):
    """Register-mode eval (bfa_eval_range, Prop 2.2): the
    full 2^n-bit DNF vector written to HBM (C4: 2^36 bits = 8 GiB) with the
    fused popcount.  Bound by the 2^n/8 bytes of stores (SURVEY §8(d):
    register eval = the count's cells + 2^n/8 bytes written)."""
    vec = torch.empty(bfa.words_for(n), dtype=torch.int64, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    for _ in range(2):
        prog.eval_range(n, 0, 1 << n, out=vec, count_out=cnt, stream=stream)
    torch.cuda.synchronize()
    launch = bfa.last_launch()
    ts = timer.run(lambda: prog.eval_range(n, 0, 1 << n, out=vec, count_out=cnt, stream=stream), steps)
    t = statistics.median(ts)
    c = int(cnt.item())
    pc = torch.zeros(1, dtype=torch.int64, device=dev)
    bfa.popcount(vec, count_out=pc, stream=stream)
    torch.cuda.synchronize()
    verified["c4_eval_count"] = c == expect and int(pc.item()) == expect
    written = (1 << n) // 8
    copy_peak, copy_src = hbm_peak()
    # the eval kernel only writes: its roofline is the store bandwidth,
    # measured here on the same 8 GiB buffer with the driver's memset
    # (torch zero_), best of 5, CUDA events on the same stream
    wt = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            a.record(stream)
            vec.zero_()
            b.record(stream)
        torch.cuda.synchronize()
        wt.append(a.elapsed_time(b) / 1e3)
    peak, src = written / min(wt), "measured store bandwidth: torch zero_ (memset) of the same 8 GiB buffer, best of 5"
    dram = traffic_for("c4_eval")
    line = {"valuations_per_s": (1 << n) / t, "ms_per_step": t * 1e3, "count": c,
            "vector_popcount": int(pc.item()), "vector_bytes": written,
            "roofline": {"bound": "hbm", "achieved": written / t / 1e9, "peak": peak / 1e9, "unit": "GB/s",
                         "frac": written / t / peak, "peak_source": src,
                         "copy_peak": copy_peak / 1e9, "frac_of_copy_peak": written / t / copy_peak,
                         "copy_peak_source": copy_src + " (read+write; a store-only stream can exceed it)",
                         "traffic": dram, "dram_frac": (dram / t / peak) if dram else None,
                         "per_unit": "2^n/8 bytes of vector stores per step, no loads"},
            "kernels": launch.get("kernels"),
            "what": "full-DNF vector of C4 (2^36 bits) in HBM + fused popcount, one register-mode eval kernel"}
    del vec
    torch.cuda.empty_cache()
    return line


def hbm_peak():
    """Measured HBM copy bandwidth (MEASURED_PEAKS.json, driver-written), else
    the profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]) * 1e9, "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    except (OSError, KeyError, ValueError):
        return 6650e9, "fallback 6.65 TB/s (B200_PROFILING.md)"


def materialised_line(bfa, torch, stream, name, steps, timer):
    """The paper's vector formulation: generator table S in
    HBM, full-vector LOP3 passes (variant 0) or fused 128-bit loads (variant
    1), popcount.  A step = one full evaluation + count."""
    cfg, variant = MATERIALISED[name]
    text, n, expect = W.config(cfg)
    prog = bfa.Program(text)
    out = torch.empty(bfa.words_for(n), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        prog.eval_materialised(n, variant, out=out, count_out=cnt, stream=stream)
    torch.cuda.synchronize()
    launch = bfa.last_launch()
    ts = timer.run(lambda: prog.eval_materialised(n, variant, out=out, count_out=cnt, stream=stream), steps)
    t = statistics.median(ts)
    vbytes = (1 << n) // 8
    fill, popc = n * vbytes, vbytes
    if variant == 0:
        logical = launch.get("logical_bytes", 0) + fill + popc
    else:
        logical = fill + (launch.get("rows_loaded", n) + 1) * vbytes + popc
    peak, src = hbm_peak()
    dram = traffic_for(name + "_step")
    line = {"valuations_per_s": (1 << n) / t, "ms_per_step": t * 1e3, "count": int(cnt.item()),
            "count_expected": expect, "workload": CONFIG_DESC[name],
            "roofline": {"bound": "hbm", "achieved": logical / t / 1e9, "peak": peak / 1e9, "unit": "GB/s",
                         "frac": logical / t / peak, "peak_source": src,
                         "traffic": dram, "dram_frac": (dram / t / peak) if dram else None,
                         "per_unit": "logical bytes = table fill n*2^n/8 + sum over passes (arity+1)*2^n/8 "
                                     "(variant 0) or (|supp|+1)*2^n/8 (variant 1) + popcount 2^n/8",
                         "logical_bytes_per_step": logical},
            "kernels": launch.get("kernels")}
    if variant == 1:
        # the fused kernel is ALU-bound for big programs: its LOP3 work per word
        luts = launch.get("luts", 0)
        line["alu"] = {"lop3_per_s": luts * (1 << (n - 5)) / t}
    return line


def run_materialised(args):
    """--config c2|c2_fused|c2_n32|c2_n32_fused as the headline (one GPU)."""
    import torch

    import paper_1310_6978_b200 as bfa
    if int(os.environ.get("WORLD_SIZE", "1")) != 1:
        raise SystemExit("materialised configs run on one GPU")
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    timer = Timer(torch, stream, "cuda")
    clocks = ClockSampler(0)
    clocks.start()
    ml = materialised_line(bfa, torch, stream, args.config, args.steps, timer)
    clk = clocks.stop()
    cfg, variant = MATERIALISED[args.config]
    text, n, _ = W.config(cfg)
    prog = bfa.Program(text)
    out = torch.empty(bfa.words_for(n), dtype=torch.int64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    host = torch.empty(out.numel(), dtype=torch.int64, pin_memory=True)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        prog.eval_materialised(n, variant, out=out, count_out=cnt, stream=stream)
        host.copy_(out, non_blocking=True)
        torch.cuda.synchronize()
    e2e = (1 << n) * args.steps / (time.perf_counter() - t0)
    line = {"metric": "valuations/s", "value": ml["valuations_per_s"], "unit": "valuations/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ml["ms_per_step"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32 (bitwise, 128-bit vector accesses)",
            "data": "synthetic (seeded generator, workloads/__init__.py)",
            "config": config_block(args.config, n, 1), "count": ml["count"], "count_expected": ml["count_expected"],
            "roofline": ml["roofline"],
            "e2e": {"value": e2e, "unit": "valuations/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": (1 << n) // 8, "call": "bfa_eval_materialised + vector D2H to pinned host"},
            "gpu_launches": (ml["kernels"] or 0) * args.steps, "clocks": clk}
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.config in MATERIALISED:
        run_materialised(args)
    else:
        run_bfa(args)


if __name__ == "__main__":
    main()
