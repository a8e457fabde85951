"""Scenario documents the control-plane golden vectors are recorded on
(test infrastructure only).

`make_doc` restates the fixture builder of the reference's own engine tests
(reference pkg/tests/test_engine.py:15-38); the variants below follow the
reference tests that pin the hot path.  The 8 reference
fixtures that fail as shipped use gpu_kv_capacity 2001 for a 2000-token
prompt; the BE start gate needs prompt + 1 + (len(ls_decode) + 256) free
(reference engine.py:587,629), so they are pinned here at 2257.
"""

from __future__ import annotations

import copy

FIXED_CAPACITY = 2257  # 2001 + the 256-token LS protect margin (engine.py:629)


def make_doc(**over) -> dict:
    doc = {
        "model": "34B",
        "policy": "omniserve",
        "horizon_s": 20,
        "seed": 4,
        "profiles": {"cluster": {"gpu_kv_capacity": 50000, "cpu_hosts": 2}},
        "engine": {"events": True, "layer_times": True},
        "workload": {
            "ls": {
                "rate": 1.5,
                "lengths": {"kind": "uniform", "prompt_min": 300, "prompt_max": 900,
                            "output_min": 30, "output_max": 90},
            },
            "be": {
                "trace": {"times": [0.0, 0.5, 1.0, 1.5, 2.0, 2.5, 3.0]},
                "lengths": {"kind": "fixed", "prompt": 2500, "output": 60},
            },
            "seed": 9,
        },
    }
    for k, v in over.items():
        doc[k] = copy.deepcopy(v)
    return doc


def offload_doc() -> dict:
    return make_doc(
        horizon_s=5,
        profiles={"cluster": {"gpu_kv_capacity": FIXED_CAPACITY, "cpu_hosts": 1}},
        workload={"be": {"trace": {"times": [0.0]},
                         "lengths": {"kind": "fixed", "prompt": 2000, "output": 6}},
                  "seed": 1},
    )


def trace_doc() -> dict:
    return make_doc(
        horizon_s=5,
        profiles={"cluster": {"gpu_kv_capacity": FIXED_CAPACITY, "cpu_hosts": 1, "layers": 4,
                              "gpu_count": 2, "tp_degree": 2}},
        engine={"events": True, "trace": True},
        workload={"be": {"trace": {"times": [0.0]},
                         "lengths": {"kind": "fixed", "prompt": 2000, "output": 6}},
                  "seed": 1},
    )


def delayed_swap_doc() -> dict:
    return make_doc(
        horizon_s=40, seed=1,
        profiles={"cluster": {"gpu_kv_capacity": 50000, "cpu_hosts": 1}},
        workload={
            "ls": {"schedule": [[0.0, 0.2], [5.0, 12.0], [12.0, 0.2]],
                   "lengths": {"kind": "fixed", "prompt": 1200, "output": 120}},
            "be": {"trace": {"times": [0.0, 0.2, 0.4, 0.6]},
                   "lengths": {"kind": "fixed", "prompt": 2000, "output": 200}},
            "seed": 5,
        },
    )


def osc_doc(delayed: bool) -> dict:
    sched, t, hi = [], 0.0, True
    while t < 30.0:
        sched.append([t, 24.0 if hi else 0.1])
        t += 0.5
        hi = not hi
    return make_doc(
        horizon_s=30, seed=2,
        profiles={"cluster": {"gpu_kv_capacity": 60000, "cpu_hosts": 1}},
        engine={"events": True, "delayed_swap_in": delayed},
        workload={
            "ls": {"schedule": sched, "lengths": {"kind": "fixed", "prompt": 600, "output": 8}},
            "be": {"trace": {"times": [0.0, 0.1, 0.2, 0.3, 0.4, 0.5]},
                   "lengths": {"kind": "fixed", "prompt": 2500, "output": 400}},
            "seed": 5,
        },
    )


def paired_doc(speed: float) -> dict:
    return make_doc(
        horizon_s=15, seed=6,
        profiles={"cluster": {"gpu_kv_capacity": 30000, "cpu_hosts": 1}},
        engine={"events": True, "layer_times": True, "cpu_speed_factor": speed},
        workload={
            "ls": {"schedule": [[0.0, 40.0], [0.25, 0.0001]],
                   "lengths": {"kind": "fixed", "prompt": 500, "output": 3000}},
            "be": {"trace": {"times": [0.0, 0.2, 0.4, 0.6]},
                   "lengths": {"kind": "fixed", "prompt": 4000, "output": 500}},
            "seed": 5,
        },
    )


# Config 1 (BASELINE.json configs[0]): tiny 2-layer model, exactly 8 LS + 32
# BE; exercises swap-out/in, injections and piggyback merges (SURVEY.md
# Appendix B).
APPENDIX_B = {
    "model": "34B", "policy": "omniserve", "horizon_s": 20, "seed": 0,
    "profiles": {
        "gpu": {"dense_base": 8.0, "dense_per_token": 0.01, "dense_tile": 128, "dense_step": 2.0,
                "attn_prefill_per_unit": 0.0005, "attn_prefill_base": 4.0,
                "attn_decode_per_unit": 0.002, "attn_decode_per_req": 0.5,
                "attn_decode_base": 3.0},
        "cluster": {"layers": 2, "gpu_count": 1, "tp_degree": 1, "cpu_hosts": 1,
                    "gpu_kv_capacity": 1000, "cpu_mem_tokens": 200000,
                    "cpu_cores_per_host": 8, "max_piggyback_per_layer": 64,
                    "merge_cost_per_result": 0.5},
    },
    "slo": {"ttft_s": 1.0, "tpot_s": 0.05},
    "engine": {"events": True, "trace": True, "layer_times": True},
    "workload": {
        "seed": 0,
        "ls": {"schedule": [[0.0, 0.0001], [1.0, 4.0], [3.0, 0.0001]],
               "lengths": {"kind": "uniform", "prompt_min": 256, "prompt_max": 512,
                           "output_min": 64, "output_max": 256}},
        "be": {"trace": {"times": [1.0 + 0.02 * i for i in range(32)]},
               "lengths": {"kind": "uniform", "prompt_min": 128, "prompt_max": 384,
                           "output_min": 64, "output_max": 256}},
    },
}


def llama8b_b200_doc(horizon_s: float = 8.0, ls_rate: float = 4.0, seed: int = 0) -> dict:
    """Config 2 shape on the virtual clock: Llama-3-8B (32 layers) on one
    B200, Poisson LS (sharegpt-like, TPOT 50 ms) + BE (longbench-like) with
    BE KV in host DRAM.  Profile coefficients are B200 roofline estimates
    for the 8B layer (weights 436 MB -> ~70 us/layer at 6.5 TB/s)."""
    return {
        "model": "34B", "policy": "omniserve", "horizon_s": horizon_s, "seed": seed,
        "profiles": {
            "gpu": {"dense_base": 70.0, "dense_per_token": 0.0, "dense_tile": 256,
                    "dense_step": 30.0, "attn_prefill_per_unit": 2.0e-5,
                    "attn_prefill_base": 3.0, "attn_decode_per_unit": 0.0007,
                    "attn_decode_per_req": 0.05, "attn_decode_base": 3.0},
            "cpu": {"attn_decode_per_unit": 0.012, "attn_decode_per_req": 2.0,
                    "attn_decode_base": 5.0},
            "cluster": {"layers": 32, "gpu_count": 1, "tp_degree": 1, "cpu_hosts": 1,
                        "gpu_kv_capacity": 60000, "cpu_mem_tokens": 1_500_000,
                        "cpu_cores_per_host": 16, "max_piggyback_per_layer": 64,
                        "merge_cost_per_result": 0.3, "pcie": [5.0, 2.0],
                        "network": [30.0, 28.0]},
        },
        "slo": {"ttft_s": 1.0, "tpot_s": 0.05},
        "engine": {"events": True, "layer_times": True},
        "workload": {
            "seed": seed,
            "ls": {"rate": ls_rate, "lengths": {"source": "sharegpt"}},
            "be": {"trace": {"rate": 2.0}, "lengths": {"source": "longbench"}},
        },
    }


SCENARIOS: dict[str, dict] = {
    "appendix_b": APPENDIX_B,
    "make_doc": make_doc(),
    "gpu_only": make_doc(policy="gpu_only"),
    "headroom": make_doc(policy="headroom", headroom_frac=0.5),
    "no_admission": make_doc(policy="no_admission_control",
                             workload={**make_doc()["workload"],
                                       "ls": {**make_doc()["workload"]["ls"], "rate": 30.0}}),
    "offload": offload_doc(),
    "trace_tp2": trace_doc(),
    "delayed_swap": delayed_swap_doc(),
    "osc_delayed": osc_doc(True),
    "osc_immediate": osc_doc(False),
    "paired_fast": paired_doc(1.0),
    "paired_slow": paired_doc(0.5),
    "noise": make_doc(horizon_s=10, engine={"events": True, "layer_times": True, "noise": True},
                      profiles={"cluster": {"gpu_kv_capacity": 50000, "cpu_hosts": 2},
                                "gpu": {"noise_rel": 0.05}, "cpu": {"noise_rel": 0.05}}),
    "llama8b_b200": llama8b_b200_doc(),
}
