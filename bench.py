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

value   = BE decode tokens emitted in the K timed iterations / device time of
          those iterations (CUDA events on the compute stream, GPU idle gaps
          between iterations included), summed over replicas / max over ranks.
e2e     = the same through the public API on the wall clock (host<->device
          metadata, token readback and PCIe piggyback traffic included).
roofline: the Dense GEMMs (dominant kernel class), algorithmic bytes per
          launch / CUDA-event time, against MEASURED_PEAKS.json HBM GB/s.
cpu_baseline: the numpy oracle port of the same step on the host cores, on a
          bounded 2-layer sample of the representative batch (scaled x16).
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
            "layers": get_transformer(args.config).n_layers, "gpu_count": 1, "tp_degree": 1, "cpu_hosts": 1,
            "gpu_kv_capacity": args.gpu_kv_tokens, "cpu_mem_tokens": 10_000_000,
            "cpu_cores_per_host": cores, "max_piggyback_per_layer": args.max_piggyback,
            "merge_cost_per_result": 0.5}},
        "slo": {"ttft_s": TTFT_SLO_S, "tpot_s": TPOT_SLO_S,
                "piggyback_reserve_us": args.piggyback_reserve_us},
        "engine": {"events": False},
        "workload": {"seed": args.seed, "ls": {"rate": ls_rate,
                                               "lengths": {"source": "sharegpt"}}},
    }


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
        spec = RequestSpec(f"BE-{i:05d}", ServiceClass.BE, p, max(o, 8), engine.now)
        r = SimRequest(spec)
        engine.requests[r.id] = r
        r.admitted = True
        r.phase = "decode"
        r.prefill_done = p
        r.tokens_out = 1
        r.token_times = [engine.now]
        r.first_token_time = engine.now
        need = r.prompt_len + r.output_len - r.tokens_out + 1
        engine.kv.alloc_host(0, need)
        r.swap_reserved = need
        r.kv_place = 0
        r.kv_held = r.ctx
        r.placement_log = [(engine.now, "cpu0")]
        slot = step.slot_of(r.id)
        step.ctx.host_kv_reserve(slot, r.prompt_len + r.output_len + 1)
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


# ----------------------------------------------------------------- CPU reference
def cpu_reference_sample(model, n_ls: int, ls_ctx: int, n_merge: int, be_ctx: int,
                         sample_layers: int = 2, steps: int = 1, warmup: int = 0) -> dict:
    """The oracle port of the serving step on the host cores (numpy fp32,
    BLAS threads = all cores): Dense over the batch + LS decode attention +
    BE piggyback attention, on `sample_layers` Llama-shaped layers, scaled to
    the full depth.  Returns per-step seconds and BE tokens/s."""
    import numpy as np

    from oracle import llama_ops as O

    rng = np.random.default_rng(0)
    d, hd, nq, nkv, ffn = model.d_model, model.head_dim, model.n_q, model.n_kv, model.ffn
    layers = []
    for _ in range(sample_layers):
        # stored [in, out] (pre-transposed) so BLAS streams each weight once
        layers.append({k: np.ascontiguousarray(
            (rng.standard_normal(shape, dtype=np.float32) * np.float32(0.02)).T)
            for k, shape in (("qkv", (model.qkv_dim, d)), ("o", (d, nq * hd)),
                             ("gu", (2 * ffn, d)), ("down", (d, ffn)))})
    # per-KV-head contiguous [2][n_kv][keys][hd] (the host layout of libhs)
    def kv_of(n):
        k = rng.standard_normal((nkv, n, hd), dtype=np.float32)
        v = rng.standard_normal((nkv, n, hd), dtype=np.float32)
        return (k, v, np.ascontiguousarray(k.transpose(0, 2, 1)))  # K^T kept for QK^T

    kv_ls = kv_of(ls_ctx)
    kv_be = kv_of(be_ctx)
    rows = n_ls + n_merge
    h = rng.standard_normal((rows, d), dtype=np.float32)

    def attend(q, kv):
        g = nq // nkv
        qh = q.reshape(nkv, g, hd)
        s = np.matmul(qh, kv[2]) / np.sqrt(hd)  # [nkv, g, keys]
        s = np.exp(s - s.max(-1, keepdims=True))
        s /= s.sum(-1, keepdims=True)
        return np.matmul(s, kv[1]).reshape(-1)

    def one_step():
        x = h
        for w in layers:
            xn = x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-5)
            qkv = xn @ w["qkv"]
            att = np.stack([attend(qkv[i, :nq * hd], kv_ls if i < n_ls else kv_be)
                            for i in range(rows)])
            x = x + att @ w["o"]
            xn = x / np.sqrt((x * x).mean(-1, keepdims=True) + 1e-5)
            gu = xn @ w["gu"]
            a = gu[:, :ffn] / (1 + np.exp(-gu[:, :ffn])) * gu[:, ffn:]
            x = x + a @ w["down"]
        return x

    for _ in range(warmup):
        one_step()
    ts = []
    for _ in range(steps):
        t = time.perf_counter()
        one_step()
        ts.append((time.perf_counter() - t) * model.n_layers / sample_layers)
    sec = statistics.median(ts)
    del O
    return {"step_s": sec, "steps": ts, "be_tokens_per_step": n_merge,
            "be_tok_s": n_merge / sec, "cores": os.cpu_count()}


# ----------------------------------------------------------------- arms
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2603_12831_b200.models import get_transformer

    model = get_transformer(args.config)
    ref = cpu_reference_sample(model, args.ref_ls_rows, 700, args.ref_merge_rows, 9000,
                               steps=args.steps, warmup=min(args.warmup, 1))
    sample = (f"numpy oracle port, {args.ref_ls_rows} LS decodes (ctx 700) + "
              f"{args.ref_merge_rows} BE piggyback merges (ctx 9000) per layer, 2 of "
              f"{model.n_layers} layers timed and scaled")
    line = {
        "impl": "reference", "metric": METRIC, "value": ref["be_tok_s"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ref["step_s"] * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "llama3-8b serving step, CPU oracle port", "model": args.config},
        "cpu_baseline": {"value": ref["be_tok_s"], "unit": UNIT, "cores": ref["cores"],
                         "kind": "port", "sample": sample},
        "e2e": {"value": ref["be_tok_s"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args) -> None:
    import numpy as np

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("gloo")

    from paper_2603_12831_b200 import profiler, replicas
    from paper_2603_12831_b200.live import LiveEngine
    from paper_2603_12831_b200.models import get_transformer
    from paper_2603_12831_b200.runtime import LiveCudaStep, RuntimeConfig
    from paper_2603_12831_b200.scenario import scenario_from_dict

    model = get_transformer(args.config)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    # the replica's CPU-attention cores: its GPU's NUMA node, split among the
    # GPUs on that node; two cores stay free for the engine thread
    cpus = replicas.core_set(local, local_world)
    workers = cpus[:-2] if len(cpus) > 3 else cpus[:1]
    cores = len(cpus)
    if args.route == "round_robin":
        # one global trace (world x the per-GPU LS rate) split over replicas
        doc = scenario_doc(args, cores, ls_rate=args.ls_rate * world)
    else:
        # independent per-replica traces (config 3: replica r uses seed + r)
        doc = scenario_doc(args, cores)
        doc["seed"] = doc["workload"]["seed"] = replicas.replica_seed(args.seed, rank)
    scenario = scenario_from_dict(doc, "bench")
    # config 5 (--workload longctx): every BE request a 32768-token prompt with
    # 136 output tokens, KV in host DRAM (4.3 GB each for Llama-3-8B)
    be_fixed = (32768, 136) if args.workload == "longctx" else None
    be_cap_tokens = (be_fixed[0] + be_fixed[1] + 64) if be_fixed else 13000 + 400
    # the pinned host KV arena of all replicas on this node must fit in RAM:
    # at most half of the available memory, split among the local replicas
    per_req = be_cap_tokens * model.kv_bytes_per_token_layer * model.n_layers
    fit = int(0.5 * replicas.mem_available_bytes() / max(local_world, 1) // per_req) - 4
    if fit < args.be_chains:
        if rank == 0:
            print(f"bench: host RAM holds {max(fit, 1)} BE requests per replica "
                  f"(asked {args.be_chains})", file=sys.stderr)
        args.be_chains = max(fit, 1)
    rt = RuntimeConfig(max_rows=args.max_rows, max_slots=512,
                       kv_pages=args.gpu_kv_tokens // 64 + 512 + 64, max_pages_per_req=256,
                       max_pos=max(16384, be_cap_tokens + 64), max_chunks=8192,
                       cpu_threads=len(workers),
                       host_kv_bytes=(args.be_chains + 4) * be_cap_tokens
                       * model.kv_bytes_per_token_layer * model.n_layers, device=local,
                       cpu_list=tuple(workers) if args.pin else ())
    t_setup = time.perf_counter()
    step = LiveCudaStep(model, rt, weight_seed=args.seed)
    models_path = ROOT / "profiles" / f"b200_{args.config}_models.json"
    if args.calibrate or not models_path.exists():
        models = profiler.calibrate(step.ctx, scenario.cluster, max_batch=args.max_rows,
                                    log=(lambda m: print(m, file=sys.stderr)) if rank == 0
                                    else None)
        if rank == 0 and args.calibrate:
            out = Path(args.calibrate_out) if args.calibrate_out else models_path
            out.parent.mkdir(parents=True, exist_ok=True)
            profiler.save(models, out, {"config": args.config, "how": "hs_probe_* on B200"})
    else:
        models = profiler.load(models_path)
    engine = LiveEngine(scenario, models=models, step=step, pace_layers=args.pace,
                        pace_tail=args.pace_tail)
    backlog = BeBacklog(engine, step, args.be_chains, args.seed + rank, fixed=be_fixed)
    if args.ls_decodes:
        prepopulate_ls(engine, step, args.ls_decodes, args.seed + rank)
    from paper_2603_12831_b200.workload import build_requests

    trace = build_requests(scenario.workload, 600.0)
    if args.route == "round_robin":
        trace = replicas.route(trace, world)[rank]
    arrivals = engine.admit_specs(trace)
    setup_s = time.perf_counter() - t_setup
    engine.t0 = time.perf_counter()
    step.set_anchor(engine.clock())
    engine.run_live(max_iterations=args.warmup, arrivals=arrivals, idle_exit=False,
                    on_iteration=backlog)
    step.ctx.sync()
    engine.drain()
    if dist:
        dist.barrier()
    launches0 = step.ctx.lib.hs_launch_count()
    h2d0, d2h0 = step.h2d_bytes, step.d2h_bytes
    cpu0, be_cpu0 = step.ctx.cpu_busy_seconds(), engine.counters["be_tokens_cpu"]
    host0 = dict(engine.host_s)
    # timed region: no per-kernel events (an event between two PDL launches
    # serialises them; measured +2.6 ms/step on llama3-8b)
    with ClockSampler(local) as clocks:
        step.ctx.sync()
        tm0 = step.ctx.timer()
        w0 = host_w0 = engine.clock()
        it0 = len(engine.iteration_log)
        engine.run_live(max_iterations=args.steps, arrivals=arrivals, idle_exit=False,
                        on_iteration=backlog)
        tm1 = step.ctx.timer()
        step.ctx.sync()
        engine.drain()
        w1 = host_w1 = engine.clock()
    if dist:
        dist.barrier()
    device_s = step.ctx.elapsed_ms(tm0, tm1) / 1e3
    launches = step.ctx.lib.hs_launch_count() - launches0
    h2d1, d2h1 = step.h2d_bytes, step.d2h_bytes
    cpu_busy = step.ctx.cpu_busy_seconds() - cpu0
    host_ms = {k: (engine.host_s[k] - host0[k]) * 1e3 / max(args.steps, 1) for k in host0}
    be_cpu = engine.counters["be_tokens_cpu"] - be_cpu0
    it1 = len(engine.iteration_log)
    # profiled window: the same workload continued for --profile-steps more
    # iterations with per-kernel-class CUDA events on the launch stream; the
    # roofline and the device breakdown come from here
    prof = (C_double * 16)()
    prof_s = 0.0
    if args.profile_steps > 0:
        step.ctx.lib.hs_profile(step.ctx.h, 1)
        step.ctx.lib.hs_profile_read(step.ctx.h, prof, 1)
        step.ctx.sync()
        tp0 = step.ctx.timer()
        engine.run_live(max_iterations=args.profile_steps, arrivals=arrivals, idle_exit=False,
                        on_iteration=backlog)
        tp1 = step.ctx.timer()
        step.ctx.sync()
        engine.drain()
        prof_s = step.ctx.elapsed_ms(tp0, tp1) / 1e3
        step.ctx.lib.hs_profile_read(step.ctx.h, prof, 1)
        step.ctx.lib.hs_profile(step.ctx.h, 0)
    iters = engine.iteration_log[it0:it1]
    # the window in engine time: from the completion of the last warm-up
    # iteration to the completion of the last timed one
    w0 = engine.iteration_log[it0 - 1]["end"] if it0 > 0 else w0
    w1 = iters[-1]["end"] if iters else w1
    m = window_metrics(engine, w0, w1)
    wall_s = host_w1 - host_w0
    stats = np.array(list(prof), dtype=np.float64).reshape(4, 4)
    # whole job: tokens, LS gaps and launches summed over replicas; device and
    # wall windows and the LS p99 maxed (the slowest replica bounds the job)
    tot, mx = replicas.aggregate(
        [m["be_tokens"], m["ls_tokens"], launches, m["ls_gaps"],
         m["tpot_attainment"] * m["ls_gaps"]],
        [device_s, wall_s, m["tpot_p99_ms"] or 0.0], dist)
    device_max, wall_max = float(mx[0]), float(mx[1])
    attain = float(tot[4] / tot[3]) if tot[3] else 1.0
    if rank != 0:
        return
    pk = peaks()
    gemm_ms, gemm_bytes, gemm_launches, gemm_flops = stats[0, 1], stats[0, 2], stats[0, 0], stats[0, 3]
    serial_gbs = gemm_bytes / (gemm_ms / 1e3) / 1e9 if gemm_ms > 0 else 0.0
    intensity = gemm_flops / gemm_bytes if gemm_bytes else 0.0
    ridge = pk["bf16_tflops"] * 1e12 / (pk["hbm_gbs"] * 1e9)
    # the roofline's launch duration: the four Dense GEMMs of all 32 layers at
    # this run's mean batch, back to back on the step stream (PDL chain intact,
    # 16 GB of weights per pass >> L2) between one CUDA event pair; per-launch
    # events (the profiled window) serialise the PDL chain and overstate it
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
                     "what": f"{args.profile_steps} profiled steps after the timed region, events "
                             "around every GEMM launch (serialises PDL; includes the LM head)",
                     "launches": int(gemm_launches), "ms_per_launch": gemm_ms / max(gemm_launches, 1),
                     "gbs": serial_gbs, "frac": serial_gbs / pk["hbm_gbs"],
                     "share_of_device_time": gemm_ms / 1e3 / max(prof_s, 1e-9)},
                 "peak_source": pk["source"],
                 "decode_attn": {"ms": stats[1, 1], "gbs": stats[1, 2] / max(stats[1, 1], 1e-9) / 1e6,
                                 "frac": stats[1, 2] / max(stats[1, 1], 1e-9) / 1e6 / pk["hbm_gbs"]}})
    value = tot[0] / device_max if device_max > 0 else 0.0
    e2e_val = tot[0] / wall_max if wall_max > 0 else 0.0
    ms_step = device_max * 1e3 / max(args.steps, 1)
    n_merges = sum(i["merges"] for i in iters)
    avg_rows = statistics.mean(i["batch_tokens"] for i in iters) if iters else 0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init weights, synthetic KV, Poisson LS trace)",
        "config": {"workload": ("llama3-8b live serving: Poisson LS (sharegpt, TPOT SLO 50 ms) + "
                                f"{args.be_chains} host-resident BE decodes kept live ("
                                + ("32768-token prompts, 136 outputs; config 5" if be_fixed
                                   else "longbench") +
                                "; completed ones replaced by new prefilled requests)"),
                   "model": args.config, "ls_rate_per_s": args.ls_rate,
                   "gpu_kv_tokens": args.gpu_kv_tokens, "max_piggyback_per_layer": args.max_piggyback,
                   "cpu_threads_per_replica": rt.cpu_threads, "parallelism": f"replicas x{world}",
                   "pace_layers": args.pace, "pace_tail": args.pace_tail,
                   "l2": "working set (16 GB weights/iteration) > 126 MB L2"},
        "ls_tpot_attainment": attain, "ls_tpot_p99_ms": float(mx[2]),
        "ls_tokens": int(tot[1]), "be_tokens": int(tot[0]), "ls_gaps": int(tot[3]),
        "slo_met": bool(attain >= 0.99),
        "merges": n_merges, "avg_batch_tokens": avg_rows,
        "batch_tokens_p90": sorted(i["batch_tokens"] for i in iters)[int(0.9 * len(iters))]
        if iters else 0,
        "be_tokens_via_cpu_attention": be_cpu,
        "cpu_pool_busy_frac": cpu_busy / max(wall_s * rt.cpu_threads, 1e-9),
        "host_ms_per_step": host_ms,
        "iteration_ms_p50": statistics.median(i["device_ms"] for i in iters
                                              if i.get("device_ms")) if iters else None,
        "device_breakdown_ms": {"window": f"{args.profile_steps} profiled steps after the timed "
                                          "region (events serialise PDL launches there)",
                                "total": prof_s * 1e3, "layers": stats[3, 1],
                                "gemm": stats[0, 1], "decode_attn": stats[1, 1],
                                "prefill_attn": stats[2, 1],
                                "other_kernels": stats[3, 1] - stats[0, 1] - stats[1, 1] - stats[2, 1],
                                "between_layers": prof_s * 1e3 - stats[3, 1]},
        "roofline": roof,
        "piggyback": {
            "ship_bytes_per_step": (d2h1 - d2h0) / max(args.steps, 1),
            "result_bytes_per_step": (h2d1 - h2d0) / max(args.steps, 1),
            "items_per_step": n_merges / max(1, len(iters)),
            "pcie_probe_64_items": pcie,
            "link_us_per_step": ((d2h1 - d2h0) / max(args.steps, 1) / (pcie["ship_sm_store_gbs"] or 1)
                                 + (h2d1 - h2d0) / max(args.steps, 1)
                                 / (pcie["result_sm_load_gbs"] or 1)) / 1e3},
        "e2e": {"value": e2e_val, "unit": UNIT,
                "h2d_bytes_per_step": (h2d1 - h2d0) / max(args.steps, 1),
                "d2h_bytes_per_step": (d2h1 - d2h0) / max(args.steps, 1)},
        "gpu_launches": int(tot[2]),
        "clocks": clocks.summary(),
        "setup_s": setup_s,
    }
    if world == 1 and not args.no_cpu_baseline:
        avg_ls = statistics.mean(i["ls_decodes"] for i in iters) if iters else 1
        avg_merge = n_merges / max(1, len(iters)) / model.n_layers
        ref = cpu_reference_sample(model, max(1, round(avg_ls)), 700, max(1, round(avg_merge)),
                                   9000, steps=1)
        line["cpu_baseline"] = {
            "value": ref["be_tok_s"], "unit": UNIT, "cores": ref["cores"], "kind": "port",
            "sample": f"numpy oracle port of this run's mean batch ({round(avg_ls)} LS decodes, "
                      f"{max(1, round(avg_merge))} piggyback merges/layer), 2 of 32 layers timed, "
                      f"scaled; {ref['step_s']:.2f} s/iteration"}
    print(json.dumps(line), flush=True)
    step.finish()


C_double = C_float = C_int = C_void_p = C_POINTER = C_byref = None


def main() -> None:
    global C_double, C_float, C_int, C_void_p, C_POINTER, C_byref
    import ctypes

    C_double, C_float, C_int = ctypes.c_double, ctypes.c_float, ctypes.c_int
    C_void_p, C_POINTER, C_byref = ctypes.c_void_p, ctypes.POINTER, ctypes.byref
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1500)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="llama3-8b")
    ap.add_argument("--workload", default="saturating", choices=["saturating", "longctx"],
                    help="BE backlog: longbench-like (config 2) or 32k-token prompts (config 5)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ls-rate", type=float, default=8.0)
    ap.add_argument("--be-chains", type=int, default=None,
                    help="host-resident BE requests kept live (default 32; 8 for --workload longctx)")
    ap.add_argument("--ls-decodes", type=int, default=0)
    ap.add_argument("--gpu-kv-tokens", type=int, default=24576)
    ap.add_argument("--max-piggyback", type=int, default=64)
    ap.add_argument("--piggyback-reserve-us", type=float, default=100.0)
    ap.add_argument("--max-rows", type=int, default=4096)
    ap.add_argument("--pace", type=int, default=2, help="layers the host may run ahead")
    ap.add_argument("--pace-tail", type=int, default=12,
                    help="final layers of an iteration launched unpaced (covers host planning)")
    ap.add_argument("--calibrate", action="store_true")
    ap.add_argument("--calibrate-out", default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--route", default="seeded", choices=["seeded", "round_robin"],
                    help="N>1: per-replica seeded traces, or one global trace routed")
    ap.add_argument("--pin", type=int, default=1, help="pin CPU-attention workers")
    ap.add_argument("--profile-steps", type=int, default=160,
                    help="profiled iterations after the timed region (roofline, breakdown)")
    ap.add_argument("--ref-ls-rows", type=int, default=8)
    ap.add_argument("--ref-merge-rows", type=int, default=16)
    args = ap.parse_args()
    if args.be_chains is None:
        args.be_chains = 8 if args.workload == "longctx" else 32
    if args.impl == "reference":
        # each CPU step is a seconds-long bounded sample: cap the count so the
        # arm finishes within minutes (the line reports the steps actually run)
        args.steps = max(1, min(args.steps, 10))
        args.warmup = min(args.warmup, 1)
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
