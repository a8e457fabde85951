#!/usr/bin/env python
"""Benchmark of the B200 OmniServe serving step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[1]): Llama-3-8B bf16 on one B200 per
replica; Poisson LS arrivals (sharegpt-like lengths, TPOT SLO 50 ms, TTFT
1 s) plus a saturating best-effort decode backlog whose KV lives in host
DRAM (longbench-like lengths, advanced by Attention Piggybacking chains on
the host CPU-attention pool).  Weights are random-init on the device; KV
contents are synthetic.  A "step" is one serving iteration of the live
engine (all 32 layers of the planned LS+BE batch plus the piggyback
exchange); the scheduler, merges, CPU service and swaps run live.

A step is one piggyback chain cycle: n_layers (32) serving iterations, the
iterations a host-resident BE request needs per token (its chain advances one
layer per iteration, reference engine.py:982-1022).  Warm-up runs W steps and
then continues until the run is stationary (>= --warmup-s of serving, chains
have completed tokens); the iterations actually used are reported.

value   = BE decode tokens emitted in the K timed steps / device time of those
          steps (CUDA events on the compute stream, GPU idle gaps between
          iterations included), summed over replicas / max over ranks.
e2e     = the same through the public API on the wall clock (host<->device
          metadata, token readback and PCIe piggyback traffic included).
roofline: the Dense GEMMs (dominant kernel class), algorithmic bytes per
          launch / CUDA-event time, against MEASURED_PEAKS.json HBM GB/s.
slo_sweep: the same workload at LS rates 1/2/4/8/16 per second (short
          windows): BE tokens/s, TPOT attainment and p99 at each rate.
cpu_baseline / --impl reference: the same serving iteration in torch bf16 on
          the host cores (oracle/torch_cpu_step.py; oneDNN/AMX GEMMs), on the
          GPU arm's mean batch composition, every layer timed.
"""

from __future__ import annotations

import argparse
import json
import os

# load every kernel at context creation: a lazily loaded module costs its
# first launch milliseconds inside the serving loop
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "BE tokens/s at >=99% LS TPOT-SLO attainment; LS p99 TPOT (ms); 1/2/4/8 B200"
UNIT = "BE tokens/s"
TPOT_SLO_S = 0.050
TTFT_SLO_S = 1.0


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        d["source"] = "measured"
        return d
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "fallback"}


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        if self.path and os.path.exists(self.path):
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------- workload
def scenario_doc(args, cores: int, ls_rate: float = None) -> dict:
    from paper_2603_12831_b200.models import get_transformer

    ls_rate = args.ls_rate if ls_rate is None else ls_rate
    return {
        "model": "34B", "policy": "omniserve", "horizon_s": 3600.0, "seed": args.seed,
        "transformer": args.config,
        "profiles": {"cluster": {
            "layers": get_transformer(args.config).n_layers, "gpu_count": 1, "tp_degree": 1,
            "cpu_hosts": 1 + getattr(args, "remote_hosts", 0),
            "gpu_kv_capacity": args.gpu_kv_tokens, "cpu_mem_tokens": 10_000_000,
            "cpu_cores_per_host": cores, "max_piggyback_per_layer": args.max_piggyback,
            "merge_cost_per_result": 0.5}},
        "slo": {"ttft_s": TTFT_SLO_S, "tpot_s": TPOT_SLO_S,
                "piggyback_reserve_us": args.piggyback_reserve_us},
        "engine": {"events": False},
        "workload": {"seed": args.seed, "ls": ls_stream(args, ls_rate),
                     **({"be": {"trace": {"rate": args.be_rate}, "lengths": be_lengths(args)}}
                        if args.be_rate > 0 else {})},
    }


def be_lengths(args) -> dict:
    """Arriving BE requests: longbench-like, or (config 5) 32768-token prompts
    with 136 outputs, prefilled on the GPU (K6) and offloaded by the policy."""
    if args.workload == "longctx":
        return {"kind": "fixed", "prompt": 32768, "output": 136}
    return {"source": "longbench"}


def ls_stream(args, ls_rate: float) -> dict:
    """Poisson LS at `ls_rate`, or (config 3) the bursty schedule of the
    reference's make_random_rate_schedule: a rate redrawn uniformly in
    [1, 8]/s every 5 s (workload.py:159-172), scaled by ls_rate / 8."""
    if args.ls_trace == "poisson":
        return {"rate": ls_rate, "lengths": {"source": "sharegpt"}}
    from paper_2603_12831_b200.workload import make_random_rate_schedule

    sched = make_random_rate_schedule(5.0, 1.0, 8.0, 600.0, args.seed)
    return {"schedule": [[t, r * ls_rate / 8.0] for t, r in sched],
            "lengths": {"source": "sharegpt"}}


def prepopulate_be(engine, step, n: int, seed: int, start: int = 0, fixed=None) -> list:
    """Saturating BE decode backlog already offloaded to host DRAM: each
    request has finished prefill (token 1 emitted) and its chain is injected
    (the state _finish_swap_out leaves, reference engine.py:437-454)."""
    from paper_2603_12831_b200.state import SimRequest
    from paper_2603_12831_b200.workload import RequestSpec, ServiceClass, longbench_like

    pairs = [fixed] if fixed else longbench_like(seed=1).pairs
    out = []
    for i in range(start, start + n):
        p, o = pairs[(seed * 7919 + i) % len(pairs)]
        spec = RequestSpec(f"BEH-{i:05d}", ServiceClass.BE, p, max(o, 8), engine.now)
        r = SimRequest(spec)
        engine.requests[r.id] = r
        r.admitted = True
        r.phase = "decode"
        r.prefill_done = p
        r.tokens_out = 1
        r.token_times = [engine.now]
        r.first_token_time = engine.now
        need = r.prompt_len + r.output_len - r.tokens_out + 1
        # --remote-hosts N: the backlog is spread evenly over the local host
        # and the N remote hosts (as if the local host's memory held 1/(N+1)
        # of it; _distribute_offload, reference engine.py:402-419)
        host = i % engine.cluster.cpu_hosts
        engine.kv.alloc_host(host, need)
        r.swap_reserved = need
        r.kv_place = host
        r.kv_held = r.ctx
        r.placement_log = [(engine.now, f"cpu{host}")]
        slot = step.slot_of(r.id)
        step.ctx.host_kv_reserve(slot, r.prompt_len + r.output_len + 1)
        if host > 0:
            # the remote host holds the request from now on; its context is as
            # synthetic as the local backlog's host KV, so none is streamed
            # (0 tokens placed: the host's region starts zeroed)
            step.ctx.cpu_place(slot, host, 0)
            step.remote_slots[slot] = host
        engine._inject(r)
        out.append(r)
    return out


class BeBacklog:
    """Keeps `n` BE requests live: every completed one is replaced by a new
    host-resident request (a stationary saturating backlog)."""

    def __init__(self, engine, step, n: int, seed: int, fixed=None):
        self.engine, self.step, self.n, self.seed, self.fixed = engine, step, n, seed, fixed
        self.next_id = n
        self.live = prepopulate_be(engine, step, n, seed, fixed=fixed)

    def __call__(self, _it: int) -> None:
        alive = [r for r in self.live if r.phase != "done"]
        short = self.n - len(alive)
        if short > 0:
            alive += prepopulate_be(self.engine, self.step, short, self.seed, self.next_id,
                                    fixed=self.fixed)
            self.next_id += short
            self.engine._dirty = True
        self.live = alive


def prepopulate_ls(engine, step, n: int, seed: int) -> list:
    """LS requests already decoding on the GPU (synthetic KV pages): a
    steady-state batch that does not depend on wall-clock arrivals (used for
    profiler captures, where kernels are serialised)."""
    from paper_2603_12831_b200.state import SimRequest
    from paper_2603_12831_b200.workload import RequestSpec, ServiceClass, sharegpt_like

    pairs = sharegpt_like().pairs
    out = []
    for i in range(n):
        p, o = pairs[(seed * 31 + i) % len(pairs)]
        r = SimRequest(RequestSpec(f"LS-P{i:04d}", ServiceClass.LS, p, max(o, 400), 0.0))
        engine.requests[r.id] = r
        r.admitted = True
        r.phase = "decode"
        r.prefill_done = p
        r.tokens_out = 1
        r.token_times = [0.0]
        r.first_token_time = 0.0
        r.kv_place = "gpu"
        r.kv_held = r.ctx
        engine.kv.alloc_gpu(r.kv_held)
        step._ensure(step.slot_of(r.id), r.ctx)
        out.append(r)
    return out


def window_metrics(engine, t0: float, t1: float) -> dict:
    from paper_2603_12831_b200.workload import ServiceClass

    be_tokens = ls_tokens = 0
    gaps = []
    for r in engine.requests.values():
        tt = r.token_times
        if r.cls == ServiceClass.BE:
            be_tokens += sum(1 for t in tt if t0 < t <= t1)
        else:
            ls_tokens += sum(1 for t in tt if t0 < t <= t1)
            gaps += [b - a for a, b in zip(tt, tt[1:]) if t0 < b <= t1]
    ok = sum(1 for g in gaps if g <= TPOT_SLO_S)
    gaps.sort()
    p99 = gaps[min(len(gaps) - 1, int(0.99 * len(gaps)))] if gaps else None
    return {"be_tokens": be_tokens, "ls_tokens": ls_tokens, "ls_gaps": len(gaps),
            "tpot_attainment": ok / len(gaps) if gaps else 1.0,
            "tpot_p99_ms": p99 * 1e3 if p99 is not None else None}


# ----------------------------------------------------------------- CPU baseline
BATCH_FILE = ROOT / "profiles" / "bench_batch.json"
DEFAULT_BATCH = {"ls_decodes": 8, "ls_ctx": 700, "be_gpu_decodes": 0, "be_gpu_ctx": 9000,
                 "merges_per_layer": 16, "merge_ctx": 9000, "chunk_tokens": 0,
                 "source": "default (no GPU-arm measurement committed)"}


def mean_batch(iters: list, n_layers: int) -> dict:
    """Mean per-iteration composition of a measured window (for the CPU
    step and the reference arm)."""
    n = max(1, len(iters))
    ls = sum(i["ls_decodes"] for i in iters)
    be = sum(i["be_gpu_decodes"] for i in iters)
    mg = sum(i["merges"] for i in iters)
    return {"ls_decodes": round(ls / n, 2), "ls_ctx": round(sum(i["ls_ctx"] for i in iters) / max(ls, 1)),
            "be_gpu_decodes": round(be / n, 2),
            "be_gpu_ctx": round(sum(i["be_gpu_ctx"] for i in iters) / max(be, 1)),
            "merges_per_layer": round(mg / n / n_layers, 2),
            "merge_ctx": round(sum(i["merge_ctx"] for i in iters) / max(mg, 1)),
            "chunk_tokens": round(sum(i["chunk_tokens"] for i in iters) / n, 1)}


def cpu_step_sample(model, batch: dict, threads: int, steps: int, warmup: int) -> dict:
    """The serving iteration on the host cores in torch bf16
    (oracle/torch_cpu_step.py) at the batch composition `batch`; every layer
    and the LM head timed.  Returns per-iteration seconds and BE tokens/s."""
    import torch

    from oracle.torch_cpu_step import TorchCpuStep

    r = lambda x: max(0, int(round(x)))  # noqa: E731
    cpu = TorchCpuStep(model, max(1, r(batch["ls_decodes"])), max(1, batch["ls_ctx"]),
                       r(batch["be_gpu_decodes"]), max(1, r(batch["merges_per_layer"])),
                       max(1, batch["merge_ctx"]), threads=threads,
                       n_prefill=r(batch.get("chunk_tokens", 0)))
    for _ in range(warmup):
        cpu.iteration()
    runs = [cpu.iteration() for _ in range(steps)]
    s = [x["s"] for x in runs]
    out = {"step_s": statistics.median(s), "steps_s": s, "be_tokens_per_step": runs[0]["be_tokens"],
           "weight_gbs": statistics.median(x["weight_gbs"] for x in runs),
           "kv_gbs": statistics.median(x["kv_gbs"] for x in runs), "threads": threads,
           "bytes_per_iteration": cpu.weight_bytes + cpu.kv_bytes}
    out["be_tok_s"] = out["be_tokens_per_step"] * len(s) / sum(s)
    del cpu, torch
    return out


def simulator_cost(args, model) -> dict:
    """The reference simulator's own cost: the virtual-time
    engine (engine.py, the bit-exact restatement of the reference's event
    loop) on this workload for a short horizon; wall seconds per simulated
    second, one core."""
    from paper_2603_12831_b200 import profiler
    from paper_2603_12831_b200.engine import Engine
    from paper_2603_12831_b200.scenario import scenario_from_dict

    doc = scenario_doc(args, 16)
    doc["horizon_s"] = 2.0
    doc["workload"]["be"] = {"trace": {"rate": 4.0}, "lengths": {"source": "longbench"}}
    path = ROOT / "profiles" / f"b200_{args.config}_models.json"
    models = profiler.load(path) if path.exists() else None
    t = time.perf_counter()
    rep = Engine(scenario_from_dict(doc, "sim"), models=models).run()
    wall = time.perf_counter() - t
    return {"wall_s_per_sim_s": wall / doc["horizon_s"], "horizon_s": doc["horizon_s"],
            "iterations": rep.counters["iterations"], "cores": 1,
            "what": "virtual-time engine (reference event loop restated bit-exactly) on this "
                    "workload (Poisson LS + longbench BE at 4/s), B200 latency models"}


def bench_config(args, model, cpu_threads: int, world: int) -> dict:
    """The workload descriptor both arms print (identical by construction)."""
    longctx = args.workload == "longctx"
    lsw = ("Poisson LS" if args.ls_trace == "poisson"
           else "bursty LS (rate redrawn in [1, 8]/s every 5 s)")
    return {"workload": (f"{args.config} live serving: {lsw} (sharegpt, TPOT SLO 50 ms) + "
                         f"{args.be_chains} host-resident BE decodes kept live ("
                         + ("32768-token prompts, 136 outputs; config 5" if longctx
                            else "longbench") +
                         "; completed ones replaced by new prefilled requests); a step is "
                         f"{model.n_layers} iterations (one piggyback chain cycle)"),
            "model": args.config, "ls_rate_per_s": args.ls_rate, "ls_trace": args.ls_trace,
            "iterations_per_step": model.n_layers,
            "gpu_kv_tokens": args.gpu_kv_tokens, "max_piggyback_per_layer": args.max_piggyback,
            "merge_decision": args.merges, "be_arrivals_per_s": args.be_rate,
            "cpu_threads_per_replica": cpu_threads, "parallelism": f"replicas x{world}",
            "l2": "working set (16 GB weights/iteration) > 126 MB L2",
            **({"cpu_hosts": 1 + args.remote_hosts} if getattr(args, "remote_hosts", 0) else {})}


def _state_summary(eng) -> dict:
    """Request states at the end of the run, counted (remote-host runs)."""
    from collections import Counter

    rep = eng.stall_report()
    cnt = Counter((rid[:2], v[0], v[1], v[2], str(v[3])) for rid, v in rep["reqs"].items())
    return {"gpu_used": rep["gpu_used"], "host_used": rep["host_used"], "pg": rep["pg"],
            "counters": {k: eng.counters[k] for k in ("ls_admitted", "swap_in_started",
                                                       "swap_in_done", "swap_out_started",
                                                       "swap_out_done", "merges")},
            "states": {"/".join(k): n for k, n in cnt.most_common(12)}}


def replica_workers(cpus: list) -> list:
    """CPU-attention workers of a replica: its cores minus two for the
    engine thread."""
    return cpus[:-2] if len(cpus) > 3 else cpus[:1]


def be_cap(args) -> int:
    """Host KV tokens reserved per BE request."""
    return 32768 + 136 + 64 if args.workload == "longctx" else 13000 + 400


def fit_be_chains(args, model, local_world: int, verbose: bool = False) -> None:
    """The pinned host KV arena of all replicas on this node must fit in RAM:
    at most half of the available memory, split among the local replicas."""
    from paper_2603_12831_b200 import replicas

    per_req = be_cap(args) * model.kv_bytes_per_token_layer * model.n_layers
    fit = int(0.5 * replicas.mem_available_bytes() / max(local_world, 1) // per_req) - 4
    if fit < args.be_chains:
        if verbose:
            print(f"bench: host RAM holds {max(fit, 1)} BE requests per replica "
                  f"(asked {args.be_chains})", file=sys.stderr)
        args.be_chains = max(fit, 1)


# ----------------------------------------------------------------- arms
def run_reference(args) -> None:
    """The reference arm: the serving iteration on the host cores (torch bf16,
    all threads), at the GPU arm's measured mean batch; a step is one
    iteration, all layers timed; exactly --steps steps after --warmup."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch

    from paper_2603_12831_b200 import replicas
    from paper_2603_12831_b200.models import get_transformer

    model = get_transformer(args.config)
    batch = json.loads(BATCH_FILE.read_text()) if BATCH_FILE.exists() else dict(DEFAULT_BATCH)
    threads = os.cpu_count() or 1
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    cpus = replicas.core_set(0, local_world)
    fit_be_chains(args, model, local_world)
    ref = cpu_step_sample(model, batch, threads, steps=args.steps, warmup=max(1, args.warmup))
    sim = simulator_cost(args, model)
    sample = (f"torch bf16 serving iteration ({threads} threads) at the GPU arm's mean batch: "
              f"{batch['ls_decodes']} LS decodes (ctx {batch['ls_ctx']}), "
              f"{batch['be_gpu_decodes']} GPU BE decodes, {batch['merges_per_layer']} piggyback "
              f"merges/layer (ctx {batch['merge_ctx']}), {batch['chunk_tokens']} prefill tokens; "
              f"all {model.n_layers} layers + LM head timed; {ref['step_s']:.2f} s/iteration, "
              f"weights {ref['weight_gbs']:.1f} GB/s, KV {ref['kv_gbs']:.1f} GB/s")
    line = {
        "impl": "reference", "metric": METRIC, "value": ref["be_tok_s"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ref["step_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(args, model, len(replica_workers(cpus)), args.gpus),
        "step": "one serving iteration on the host cores (a bounded sample of the workload)",
        "cpu_baseline": {"value": ref["be_tok_s"], "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": sample},
        "batch": batch, "steps_s": ref["steps_s"],
        "simulator": sim,
        "e2e": {"value": ref["be_tok_s"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    del torch


class Replica:
    """One GPU replica: context, engine, BE backlog and trace."""

    def __init__(self, args, world: int, rank: int, local: int, local_world: int,
                 model=None, make_ctx=None, device=None):
        from paper_2603_12831_b200 import profiler, replicas
        from paper_2603_12831_b200.models import get_transformer
        from paper_2603_12831_b200.runtime import LiveCudaStep

        self.args, self.world, self.rank = args, world, rank
        model = self.model = model or get_transformer(args.config)
        # the replica's CPU-attention cores: its GPU's NUMA node, split among the
        # GPUs on that node; two cores stay free for the engine thread
        cpus = replicas.core_set(local, local_world)
        workers = replica_workers(cpus)
        self.cores = len(cpus)
        self.be_fixed = (32768, 136) if args.workload == "longctx" else None
        fit_be_chains(args, model, local_world, verbose=rank == 0)
        rt = self.rt = _replica_rt(args, model, local, local_world, device)
        self.remote = None
        if args.remote_hosts:
            # remote CPU hosts: separate processes on the cores
            # outside this replica's set (the other NUMA node), reached over TCP
            from paper_2603_12831_b200 import cpu_host

            others = sorted(set(os.sched_getaffinity(0)) - set(cpus))
            k = args.remote_hosts
            per = len(others) // k
            sets = [others[i * per:(i + 1) * per] for i in range(k)] if per else None
            self.remote = cpu_host.RemoteHosts(model, k, threads=max(1, per or 2),
                                               max_slots=rt.max_slots, cpu_sets=sets)
            import atexit

            atexit.register(self.remote.close)
            rt.remote_hosts = tuple((h.addr, h.port) for h in self.remote.hosts)
            self.remote_threads = [max(1, per or 2)] * k
        # make_ctx (a TP group's rank 0): the caller builds the context -- the
        # shard, the group's exchange and shared tags -- and mirrors it
        self.step = LiveCudaStep(model, rt, weight_seed=args.seed,
                                 device_merges=args.merges == "device",
                                 ctx=make_ctx(rt) if make_ctx else None)
        models_path = ROOT / "profiles" / f"b200_{args.config}_models.json"
        scen = self.scenario(args.ls_rate)
        if make_ctx and not models_path.exists():
            # a TP shard cannot run the profiler's probes alone (the fused
            # all-reduce needs every rank); use the unsharded model's fit
            models_path = ROOT / "profiles" / "b200_llama3-8b_models.json"
        if not make_ctx and (args.calibrate or not models_path.exists()):
            self.models = profiler.calibrate(
                self.step.ctx, scen.cluster, max_batch=args.max_rows,
                log=(lambda m: print(m, file=sys.stderr)) if rank == 0 else None)
            if rank == 0 and args.calibrate:
                out = Path(args.calibrate_out) if args.calibrate_out else models_path
                out.parent.mkdir(parents=True, exist_ok=True)
                profiler.save(self.models, out, {"config": args.config, "how": "hs_probe_* on B200"})
        else:
            self.models = profiler.load(models_path)

    def scenario(self, ls_rate: float):
        from paper_2603_12831_b200 import replicas
        from paper_2603_12831_b200.scenario import scenario_from_dict

        args = self.args
        if args.route == "round_robin":
            # one global trace (world x the per-GPU LS rate) split over replicas
            doc = scenario_doc(args, self.cores, ls_rate=ls_rate * self.world)
        else:
            # independent per-replica traces (config 3: replica r uses seed + r)
            doc = scenario_doc(args, self.cores, ls_rate=ls_rate)
            doc["seed"] = doc["workload"]["seed"] = replicas.replica_seed(args.seed, self.rank)
        return scenario_from_dict(doc, "bench")

    def start(self, ls_rate: float):
        """A fresh engine on the (reset) context: BE backlog + LS trace."""
        from paper_2603_12831_b200 import replicas
        from paper_2603_12831_b200.live import LiveEngine
        from paper_2603_12831_b200.workload import build_requests

        args = self.args
        scen = self.scenario(ls_rate)
        eng = self.engine = LiveEngine(scen, models=self.models, step=self.step,
                                       pace_layers=args.pace, pace_tail=args.pace_tail)
        self.backlog = BeBacklog(eng, self.step, args.be_chains, args.seed + self.rank,
                                 fixed=self.be_fixed)
        if args.ls_decodes:
            prepopulate_ls(eng, self.step, args.ls_decodes, args.seed + self.rank)
        trace = build_requests(scen.workload, 600.0)
        if args.route == "round_robin":
            trace = replicas.route(trace, self.world)[self.rank]
        self.arrivals = eng.admit_specs(trace)
        eng.t0 = time.perf_counter()
        self.step.set_anchor(eng.clock())
        return eng

    def run(self, iterations: int) -> int:
        return self.engine.run_live(max_iterations=iterations, arrivals=self.arrivals,
                                    idle_exit=False, on_iteration=self.backlog)

    def warm(self, min_iters: int, min_s: float, max_iters: int) -> int:
        """Warm-up to a stationary state: at least `min_iters` iterations and
        `min_s` seconds of serving, and at least one BE token completed
        through Attention Piggybacking (chains in flight everywhere)."""
        eng, L = self.engine, self.model.n_layers
        n = self.run(min_iters)
        while n < max_iters and (eng.clock() < min_s or eng.counters["be_tokens_cpu"] == 0):
            n += self.run(L)
        self.step.ctx.sync()
        eng.drain()
        return n


def timed_window(rep, iterations: int, dist) -> dict:
    """Run `iterations` serving iterations between two device events on the
    compute stream; per-replica measurements of the window."""
    eng, step = rep.engine, rep.step
    if dist:
        dist.barrier()
    launches0 = step.ctx.lib.hs_launch_count()
    h2d0, d2h0 = step.h2d_bytes, step.d2h_bytes
    cpu0, be_cpu0 = step.ctx.cpu_busy_seconds(), eng.counters["be_tokens_cpu"]
    host0 = dict(eng.host_s)
    step.ctx.sync()
    tm0 = step.ctx.timer()
    w0 = eng.clock()
    it0 = len(eng.iteration_log)
    rep.run(iterations)
    tm1 = step.ctx.timer()
    step.ctx.sync()
    eng.drain()
    w1 = eng.clock()
    if dist:
        dist.barrier()
    iters = eng.iteration_log[it0:]
    # the window in engine time: from the completion of the last warm-up
    # iteration to the completion of the last timed one
    e0 = eng.iteration_log[it0 - 1]["end"] if it0 > 0 else w0
    e1 = iters[-1]["end"] if iters else w1
    m = window_metrics(eng, e0, e1)
    m.update({"device_s": step.ctx.elapsed_ms(tm0, tm1) / 1e3, "wall_s": w1 - w0,
              "launches": step.ctx.lib.hs_launch_count() - launches0,
              "h2d": step.h2d_bytes - h2d0, "d2h": step.d2h_bytes - d2h0,
              "cpu_busy": step.ctx.cpu_busy_seconds() - cpu0,
              "be_cpu": eng.counters["be_tokens_cpu"] - be_cpu0,
              "host_s": {k: eng.host_s[k] - host0[k] for k in host0}, "iters": iters})
    return m


def run_tp(args) -> None:
    """Config 4: one tensor-parallel group over all ranks of the job (one
    process per GPU).  Rank 0 plans and serves through a MirrorContext; the
    other ranks replay its calls on their shards (tp.follow); the fused
    all-reduce runs over P2P / NVLink and the ranks agree on every merge
    through shared completion tags (device-polled merges)."""
    import torch
    import torch.distributed as dist

    from paper_2603_12831_b200 import tp
    from paper_2603_12831_b200.models import get_transformer
    from paper_2603_12831_b200.runtime import HsContext

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.tp:
        raise SystemExit(f"bench: --tp {args.tp} needs WORLD_SIZE {args.tp} (got {world})")
    if args.merges != "device":
        raise SystemExit("bench: a live TP group needs --merges device (merge agreement)")
    # a group larger than the box (a functional run) time-shares its GPUs
    dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    shard = tp.shard_config(get_transformer(args.config), world)
    prefix = f"/hs_bench_tp_{os.environ.get('MASTER_PORT', '0')}"
    ctx_box = {}

    def make_ctx(rt):
        ctx = HsContext(shard, rt)
        ctx.init_weights(args.seed * 131 + rank)  # random-init shard of each rank
        tp.open_group(ctx, rank, world)
        ctx.pg_enable(True)
        tp.share_tags(ctx, rank, world, prefix)
        ctx_box["ctx"] = ctx
        return tp.MirrorContext(ctx) if rank == 0 else ctx

    args.pace, args.pace_tail = 64, 0  # unpaced: the followers get one message per iteration
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    if rank != 0:
        # the same runtime sizes as rank 0's replica
        rt = _replica_rt(argparse.Namespace(**vars(args)), shard, local, local_world, dev)
        ctx = make_ctx(rt)
        tp.follow(ctx)
        dist.barrier()
        return
    rep = Replica(args, 1, 0, local, local_world, model=shard, make_ctx=make_ctx, device=dev)
    L = shard.n_layers
    rep.start(args.ls_rate)
    warm = rep.warm(args.warmup * L, args.warmup_s, max(args.warmup, 40) * L)
    with ClockSampler(dev) as clocks:
        m = timed_window(rep, args.steps * L, None)
    rep.step.finish()
    rep.step.ctx.flush(stop=True)
    dist.barrier()
    iters = m["iters"]
    line = {
        "metric": METRIC, "value": m["be_tokens"] / m["device_s"] if m["device_s"] else 0.0,
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": m["device_s"] * 1e3 / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weight shards, synthetic KV, Poisson LS trace)",
        "config": dict(bench_config(args, shard, rep.rt.cpu_threads, 1),
                       parallelism=f"tp{world} (one group, live, device-decided merges)"),
        "iterations_timed": len(iters), "warmup_iterations": warm,
        "ls_tpot_attainment": m["tpot_attainment"], "ls_tpot_p99_ms": m["tpot_p99_ms"],
        "be_tokens": m["be_tokens"], "ls_gaps": m["ls_gaps"],
        "be_tokens_via_cpu_attention": m["be_cpu"],
        "iteration_ms_p50": statistics.median(i["device_ms"] for i in iters
                                              if i.get("device_ms")) if iters else None,
        "e2e": {"value": m["be_tokens"] / m["wall_s"] if m["wall_s"] else 0.0, "unit": UNIT,
                "h2d_bytes_per_step": m["h2d"] / max(args.steps, 1),
                "d2h_bytes_per_step": m["d2h"] / max(args.steps, 1)},
        "gpu_launches": int(m["launches"]), "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)


def _replica_rt(args, model, local: int, local_world: int, device=None):
    """The RuntimeConfig Replica builds for `model` (TP followers need the
    same sizes as rank 0 without building an engine)."""
    from paper_2603_12831_b200 import replicas
    from paper_2603_12831_b200.runtime import RuntimeConfig

    cpus = replicas.core_set(local, local_world)
    workers = replica_workers(cpus)
    fit_be_chains(args, model, local_world)
    cap = be_cap(args)
    return RuntimeConfig(
        max_rows=args.max_rows, max_slots=512, kv_pages=args.gpu_kv_tokens // 64 + 512 + 64,
        max_pages_per_req=max(256, (cap + 127) // 64), max_pos=max(16384, cap + 64),
        max_chunks=8192, cpu_threads=len(workers),
        host_kv_bytes=(args.be_chains + 4) * cap * model.kv_bytes_per_token_layer * model.n_layers,
        device=local if device is None else device, cpu_list=tuple(workers) if args.pin else ())


def run_ours(args) -> None:
    import numpy as np

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    import torch

    # ranks beyond the box's GPUs time-share them (a functional multi-rank
    # run on a smaller box; gpus_active reports the distinct devices)
    n_dev = max(1, torch.cuda.device_count())
    dev = local % n_dev
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(dev)
        dist.init_process_group("gloo")
        if world != args.gpus:
            raise SystemExit(f"bench: WORLD_SIZE {world} != --gpus {args.gpus}")

    from paper_2603_12831_b200 import replicas

    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    t_setup = time.perf_counter()
    rep = Replica(args, world, rank, local, local_world, device=dev)
    model, step = rep.model, rep.step
    L = model.n_layers
    rep.start(args.ls_rate)
    setup_s = time.perf_counter() - t_setup
    warm_iters = rep.warm(args.warmup * L, args.warmup_s, max(args.warmup, 40) * L)
    with ClockSampler(dev) as clocks:
        m = timed_window(rep, args.steps * L, dist)
    eng = rep.engine
    iters = m["iters"]
    # profiled window: the same workload continued for --profile-steps more
    # iterations with per-kernel-class CUDA events on the launch stream (the
    # device breakdown; events serialise the PDL chain there)
    prof = (C_double * 16)()
    prof_s = 0.0
    if args.profile_steps > 0:
        step.ctx.lib.hs_profile(step.ctx.h, 1)
        step.ctx.lib.hs_profile_read(step.ctx.h, prof, 1)
        step.ctx.sync()
        tp0 = step.ctx.timer()
        rep.run(args.profile_steps)
        tp1 = step.ctx.timer()
        step.ctx.sync()
        eng.drain()
        prof_s = step.ctx.elapsed_ms(tp0, tp1) / 1e3
        step.ctx.lib.hs_profile_read(step.ctx.h, prof, 1)
        step.ctx.lib.hs_profile(step.ctx.h, 0)
    stats = np.array(list(prof), dtype=np.float64).reshape(4, 4)
    # whole job: tokens, LS gaps and launches summed over replicas; device and
    # wall windows and the LS p99 maxed (the slowest replica bounds the job)
    tot, mx = replicas.aggregate(
        [m["be_tokens"], m["ls_tokens"], m["launches"], m["ls_gaps"],
         m["tpot_attainment"] * m["ls_gaps"], m["be_cpu"], 1.0],
        [m["device_s"], m["wall_s"], m["tpot_p99_ms"] or 0.0], dist)
    device_max, wall_max = float(mx[0]), float(mx[1])
    attain = float(tot[4] / tot[3]) if tot[3] else 1.0
    roof, pcie = roofline_and_link(args, rep, iters, stats, prof_s)
    batch = mean_batch(iters, L)
    # LS-rate sweep (short windows on the same context)
    sweep = []
    if args.sweep:
        for lam in args.sweep:
            step.reset()
            rep.start(lam)
            rep.warm(args.sweep_warmup * L, args.warmup_s, max(args.sweep_warmup, 20) * L)
            ms = timed_window(rep, args.sweep_steps * L, dist)
            t2, m2 = replicas.aggregate([ms["be_tokens"], ms["ls_gaps"],
                                         ms["tpot_attainment"] * ms["ls_gaps"]],
                                        [ms["device_s"], ms["tpot_p99_ms"] or 0.0], dist)
            att = float(t2[2] / t2[1]) if t2[1] else 1.0
            sweep.append({"ls_rate_per_s": lam, "be_tok_s": float(t2[0] / m2[0]) if m2[0] else 0.0,
                          "tpot_attainment": att, "tpot_p99_ms": float(m2[1]),
                          "ls_gaps": int(t2[1]), "slo_met": bool(att >= 0.99),
                          "ms_per_iteration": float(m2[0]) * 1e3 / max(1, len(ms["iters"]))})
    if rank != 0:
        step.finish()
        return
    value = tot[0] / device_max if device_max > 0 else 0.0
    e2e_val = tot[0] / wall_max if wall_max > 0 else 0.0
    ms_step = device_max * 1e3 / max(args.steps, 1)
    n_merges = sum(i["merges"] for i in iters)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, synthetic KV, Poisson LS trace)",
        "config": bench_config(args, model, rep.rt.cpu_threads, world),
        "iterations_timed": len(iters), "warmup_iterations": warm_iters,
        **({"remote_hosts": {"n": args.remote_hosts, "threads": rep.remote_threads,
                             "engine_state": _state_summary(eng),
                             "per_host": [step.ctx.remote_stats(h)
                                          for h in range(1, args.remote_hosts + 1)]}}
           if rep.remote else {}),
        "gpus_active": int(min(tot[6], n_dev * (world // max(1, local_world)))),
        "gpus_time_shared": bool(local_world > n_dev),
        "be_prefill_tok_s": (sum(i.get("be_chunk_tokens", 0) for i in iters) * world
                             / device_max) if device_max > 0 else 0.0,
        "ls_tpot_attainment": attain, "ls_tpot_p99_ms": float(mx[2]),
        "ls_tokens": int(tot[1]), "be_tokens": int(tot[0]), "ls_gaps": int(tot[3]),
        "slo_met": bool(attain >= 0.99),
        "merges": n_merges, "avg_batch_tokens": statistics.mean(i["batch_tokens"] for i in iters)
        if iters else 0,
        "batch_tokens_p90": sorted(i["batch_tokens"] for i in iters)[int(0.9 * len(iters))]
        if iters else 0,
        "batch": batch,
        "be_tokens_via_cpu_attention": int(tot[5]),
        "cpu_pool_busy_frac": m["cpu_busy"] / max(m["wall_s"] * rep.rt.cpu_threads, 1e-9),
        "host_ms_per_iteration": {k: v * 1e3 / max(1, len(iters)) for k, v in m["host_s"].items()},
        "iteration_ms_p50": statistics.median(i["device_ms"] for i in iters
                                              if i.get("device_ms")) if iters else None,
        "device_breakdown_ms": {"window": f"{args.profile_steps} profiled iterations after the "
                                          "timed region (events serialise PDL launches there)",
                                "total": prof_s * 1e3, "layers": stats[3, 1],
                                "gemm": stats[0, 1], "decode_attn": stats[1, 1],
                                "prefill_attn": stats[2, 1],
                                "other_kernels": stats[3, 1] - stats[0, 1] - stats[1, 1] - stats[2, 1],
                                "between_layers": prof_s * 1e3 - stats[3, 1]},
        "roofline": roof,
        "piggyback": {
            "ship_bytes_per_iteration": m["d2h"] / max(1, len(iters)),
            "result_bytes_per_iteration": m["h2d"] / max(1, len(iters)),
            "items_per_iteration": n_merges / max(1, len(iters)),
            "pcie_probe_64_items": pcie},
        "e2e": {"value": e2e_val, "unit": UNIT,
                "h2d_bytes_per_step": m["h2d"] / max(args.steps, 1),
                "d2h_bytes_per_step": m["d2h"] / max(args.steps, 1)},
        "gpu_launches": int(tot[2]),
        "clocks": clocks.summary(),
        "setup_s": setup_s,
    }
    if sweep:
        ok = [s_ for s_ in sweep if s_["slo_met"]]
        line["slo_sweep"] = sweep
        line["slo_sweep_window"] = (f"{args.sweep_steps} steps per rate after >= {args.warmup_s} s "
                                    "of warm-up, same context")
        line["max_be_tok_s_at_slo"] = max((s_["be_tok_s"] for s_ in ok), default=None)
    step.finish()
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        ref = cpu_step_sample(model, batch, threads, steps=1, warmup=1)
        line["cpu_baseline"] = {
            "value": ref["be_tok_s"], "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"torch bf16 serving iteration on the host cores at this run's mean batch "
                      f"({batch['ls_decodes']} LS decodes, {batch['merges_per_layer']} piggyback "
                      f"merges/layer, {batch['chunk_tokens']} prefill tokens), every layer timed; "
                      f"{ref['step_s']:.2f} s/iteration, weights {ref['weight_gbs']:.1f} GB/s"}
    print(json.dumps(line), flush=True)
    if args.write_batch:
        BATCH_FILE.write_text(json.dumps({**batch, "source": f"bench.py GPU arm, {len(iters)} "
                                          "timed iterations"}, indent=1) + "\n")


def roofline_and_link(args, rep, iters, stats, prof_s):
    """Dense-GEMM roofline at the run's mean batch (in-stream, PDL chain
    intact) and the PCIe rate of the piggyback mailboxes."""
    step, model = rep.step, rep.model
    pk = peaks()
    gemm_ms, gemm_bytes, gemm_launches = stats[0, 1], stats[0, 2], stats[0, 0]
    serial_gbs = gemm_bytes / (gemm_ms / 1e3) / 1e9 if gemm_ms > 0 else 0.0
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    rows_mean = max(1, round(statistics.mean(i["batch_tokens"] for i in iters))) if iters else 1
    us_l, by_l = C_float(), C_double()
    step.ctx.lib.hs_probe_gemm_stream.argtypes = [C_void_p, C_int, C_int, C_POINTER(C_float),
                                                 C_POINTER(C_double)]
    rc = step.ctx.lib.hs_probe_gemm_stream(step.ctx.h, rows_mean, 5, C_byref(us_l), C_byref(by_l))
    if rc != 0:
        raise RuntimeError(f"hs_probe_gemm_stream failed ({rc})")
    gemm_us, gemm_by = us_l.value, by_l.value
    achieved_gbs = gemm_by / (gemm_us * 1e-6) / 1e9
    # PCIe rate of the piggyback mailboxes (q|k|v ship D2H by SM stores into
    # mapped pinned memory, host results H2D by SM loads), with the copy
    # engine's rate for the same bytes alongside
    step.ctx.lib.hs_probe_pcie.argtypes = [C_void_p, C_int, C_int, C_int, C_POINTER(C_float),
                                          C_POINTER(C_double)]
    pcie = {}
    for d_, name in enumerate(("ship_sm_store", "result_sm_load", "copy_engine_d2h",
                               "copy_engine_h2d")):
        rc = step.ctx.lib.hs_probe_pcie(step.ctx.h, d_, 64, 7, C_byref(us_l), C_byref(by_l))
        pcie[name + "_gbs"] = by_l.value / (us_l.value * 1e-6) / 1e9 if rc == 0 else None
    params = (model.qkv_dim * model.d_model + model.d_model * model.n_q * model.head_dim
              + 3 * model.ffn * model.d_model)
    flops_l = 2.0 * rows_mean * params / 4
    intensity = flops_l / gemm_by
    traffic = None
    tr_path = ROOT / "profiles" / "ncu_gemm_traffic.json"
    if tr_path.exists():
        traffic = json.loads(tr_path.read_text()).get("dram_bytes_per_launch")
    if intensity < ridge:
        roof = {"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved_gbs / pk["hbm_gbs"], "traffic": traffic}
    else:
        tf = flops_l / (gemm_us * 1e-6) / 1e12
        roof = {"bound": "tensor", "achieved": tf, "peak": pk["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": tf / pk["bf16_tflops_sustained"], "traffic": traffic}
    roof.update({"kernel": "gemm_bf16_tn_kernel (tcgen05, Dense QKV/O/gate-up/down)",
                 "rows": rows_mean, "us_per_launch": gemm_us, "bytes_per_launch": gemm_by,
                 "window": f"4 x {model.n_layers} Dense GEMM launches at the run's mean batch "
                           f"({rows_mean} rows) back to back between one event pair (median of 5)",
                 "serialised_window": {
                     "what": f"{args.profile_steps} profiled iterations after the timed region, "
                             "events around every GEMM launch (serialises PDL; includes the LM head)",
                     "launches": int(gemm_launches), "ms_per_launch": gemm_ms / max(gemm_launches, 1),
                     "gbs": serial_gbs, "frac": serial_gbs / pk["hbm_gbs"],
                     "share_of_device_time": gemm_ms / 1e3 / max(prof_s, 1e-9)},
                 "peak_source": pk["source"],
                 "decode_attn": {"ms": stats[1, 1], "gbs": stats[1, 2] / max(stats[1, 1], 1e-9) / 1e6,
                                 "frac": stats[1, 2] / max(stats[1, 1], 1e-9) / 1e6 / pk["hbm_gbs"]}})
    return roof, pcie


C_double = C_float = C_int = C_void_p = C_POINTER = C_byref = None


def spawn_replicas(n: int) -> int:
    """`--gpus N` outside torchrun: one replica process per GPU via
    torch.distributed.run (rank 0 prints the line)."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())]
    return subprocess.call(cmd + sys.argv[1:])


def main() -> None:
    global C_double, C_float, C_int, C_void_p, C_POINTER, C_byref
    import ctypes

    C_double, C_float, C_int = ctypes.c_double, ctypes.c_float, ctypes.c_int
    C_void_p, C_POINTER, C_byref = ctypes.c_void_p, ctypes.POINTER, ctypes.byref
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--tp", type=int, default=1,
                    help="config 4: all ranks form one tensor-parallel group (live, one planner)")
    ap.add_argument("--steps", type=int, default=40, help="timed steps (chain cycles)")
    ap.add_argument("--warmup", type=int, default=8, help="warm-up steps (at least)")
    ap.add_argument("--warmup-s", type=float, default=2.0,
                    help="minimum seconds of serving before the timed region (LS ramp)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--workload", default="saturating", choices=["saturating", "longctx"],
                    help="BE backlog: longbench-like (config 2) or 32k-token prompts (config 5)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ls-rate", type=float, default=8.0)
    ap.add_argument("--ls-trace", default="poisson", choices=["poisson", "burst"],
                    help="LS arrivals: Poisson at --ls-rate, or the bursty 5 s schedule of "
                         "config 3 (peak --ls-rate)")
    ap.add_argument("--sweep", type=lambda s: [float(x) for x in s.split(",") if x],
                    default=[1.0, 2.0, 4.0, 8.0, 16.0],
                    help="LS rates of the SLO sweep (empty string: none)")
    ap.add_argument("--sweep-steps", type=int, default=4)
    ap.add_argument("--sweep-warmup", type=int, default=2)
    ap.add_argument("--be-chains", type=int, default=None,
                    help="host-resident BE requests kept live (default 32; 8 for --workload longctx)")
    ap.add_argument("--ls-decodes", type=int, default=0)
    ap.add_argument("--be-rate", type=float, default=None,
                    help="BE arrivals per second, prefilled on the GPU and offloaded by the "
                         "policy, on top of the host-resident decode backlog (default 0; "
                         "0.25 with --workload longctx: 32k-token prompts)")
    ap.add_argument("--gpu-kv-tokens", type=int, default=24576)
    ap.add_argument("--max-piggyback", type=int, default=64)
    ap.add_argument("--piggyback-reserve-us", type=float, default=100.0)
    ap.add_argument("--max-rows", type=int, default=4096)
    ap.add_argument("--pace", type=int, default=None,
                    help="layers the host may run ahead of the GPU (default 2)")
    ap.add_argument("--pace-tail", type=int, default=None,
                    help="final layers of an iteration launched unpaced (covers host planning; "
                         "default 12)")
    ap.add_argument("--merges", default="device", choices=["device", "host"],
                    help="piggyback merge decision: GPU controller polling the completion "
                         "tags (csrc/piggyback.cu), or the host at each layer launch")
    ap.add_argument("--calibrate", action="store_true")
    ap.add_argument("--calibrate-out", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--write-batch", action="store_true",
                    help="record the measured mean batch for the reference arm")
    ap.add_argument("--route", default="seeded", choices=["seeded", "round_robin"],
                    help="N>1: per-replica seeded traces, or one global trace routed")
    ap.add_argument("--pin", type=int, default=1, help="pin CPU-attention workers")
    ap.add_argument("--remote-hosts", type=int, default=0,
                    help="remote CPU hosts (cpu_host processes on the other cores, over TCP); "
                         "the BE backlog is spread over the local and remote hosts")
    ap.add_argument("--profile-steps", type=int, default=160,
                    help="profiled iterations after the timed region (device breakdown)")
    args = ap.parse_args()
    if args.be_chains is None:
        args.be_chains = 8 if args.workload == "longctx" else 32
    # launch pacing: with host-decided merges it bounds their freshness; with
    # device-decided ones it only keeps the GPU queue short (measured: the
    # unpaced device-merge run was 5 % slower per step, 175 vs 166 ms)
    if args.pace is None:
        args.pace = 2
    if args.pace_tail is None:
        args.pace_tail = 12
    if args.be_rate is None:
        args.be_rate = 0.25 if args.workload == "longctx" else 0.0
    if args.workload == "longctx" and args.gpu_kv_tokens == 24576:
        # a 32k-token prompt is prefilled on the GPU: room for one next to
        # the LS envelope (the policy offloads it after prefill)
        args.gpu_kv_tokens = 45056
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_replicas(args.gpus))
    if args.impl == "reference":
        run_reference(args)
    elif args.tp > 1:
        run_tp(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
