"""Independent replicas: NUMA core sets,
the trace router, and the N>1 bench path exercised with world_size-2 gloo
process groups on CPU (one rank per replica, no data-path collective; only
the end-of-run reduction crosses ranks)."""

from __future__ import annotations

import copy
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.scenarios import make_doc
from paper_2603_12831_b200 import replicas
from paper_2603_12831_b200.engine import Engine
from paper_2603_12831_b200.scenario import scenario_from_dict
from paper_2603_12831_b200.workload import ServiceClass, build_requests


# ----------------------------------------------------------------- topology
def _fake_sysfs(root, nodes: int, cores_per_node: int, smt: int = 2):
    """Two-socket-style layout: node n owns physical cores
    [n*cpn, (n+1)*cpn); the SMT sibling of cpu c is c + nodes*cpn."""
    total_phys = nodes * cores_per_node
    for n in range(nodes):
        cpus = [c for c in range(n * cores_per_node, (n + 1) * cores_per_node)]
        sib = [c + total_phys * s for s in range(1, smt) for c in cpus]
        d = root / f"devices/system/node/node{n}"
        d.mkdir(parents=True)
        (d / "cpulist").write_text(",".join(str(c) for c in sorted(cpus + sib)) + "\n")
    for c in range(total_phys):
        group = [c + total_phys * s for s in range(smt)]
        for x in group:
            t = root / f"devices/system/cpu/cpu{x}/topology"
            t.mkdir(parents=True)
            t.joinpath("thread_siblings_list").write_text(",".join(map(str, group)) + "\n")
    return list(range(total_phys * smt))


def test_parse_cpulist():
    assert replicas.parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert replicas.parse_cpulist("") == []


def test_core_sets_are_numa_local_disjoint_and_keep_siblings(tmp_path):
    allowed = _fake_sysfs(tmp_path, nodes=2, cores_per_node=8)
    gpu_nodes = [0, 0, 0, 0, 1, 1, 1, 1]
    sets = [replicas.core_set(r, 8, gpu_nodes, allowed, tmp_path) for r in range(8)]
    seen = set()
    for r, cs in enumerate(sets):
        assert len(cs) == 4  # 2 physical cores x 2 threads
        assert not seen & set(cs)
        seen |= set(cs)
        node = gpu_nodes[r]
        node_cpus = set(replicas.node_cpus(node, tmp_path))
        assert set(cs) <= node_cpus
        phys = [c for c in cs if c < 16]
        assert sorted(cs) == sorted(phys + [c + 16 for c in phys])  # siblings together
    assert seen == set(allowed)


def test_core_set_unknown_node_splits_allowed(tmp_path):
    allowed = list(range(12))
    sets = [replicas.core_set(r, 3, [-1, -1, -1], allowed, tmp_path) for r in range(3)]
    assert sets == [[0, 1, 2, 3], [4, 5, 6, 7], [8, 9, 10, 11]]
    with pytest.raises(ValueError):
        replicas.core_set(3, 3, [-1, -1, -1], allowed, tmp_path)


def test_core_set_respects_cgroup_allowance(tmp_path):
    _fake_sysfs(tmp_path, nodes=2, cores_per_node=8)
    allowed = list(range(4)) + list(range(16, 20))  # 4 cores of node 0 (+ siblings)
    cs = replicas.core_set(0, 2, [0, 0], allowed, tmp_path)
    assert cs == [0, 1, 16, 17]


# ----------------------------------------------------------------- router
def _trace(ls_rate=6.0, horizon=6.0):
    doc = make_doc(horizon_s=horizon)
    doc["workload"]["ls"]["rate"] = ls_rate
    return build_requests(scenario_from_dict(doc, "r").workload, horizon), doc


@pytest.mark.parametrize("n", [1, 2, 3, 8])
def test_route_is_disjoint_covering_balanced_and_ordered(n):
    specs, _ = _trace()
    parts = replicas.route(specs, n)
    assert len(parts) == n
    flat = [s.id for p in parts for s in p]
    assert sorted(flat) == sorted(s.id for s in specs)
    assert len(set(flat)) == len(flat)
    for cls in (ServiceClass.LS, ServiceClass.BE):
        counts = [sum(1 for s in p if s.cls == cls) for p in parts]
        assert max(counts) - min(counts) <= 1
    for p in parts:
        keys = [(s.arrival_time, s.cls.value, s.id) for s in p]
        assert keys == sorted(keys)
    with pytest.raises(ValueError):
        replicas.route(specs, 0)


def test_aggregate_without_process_group():
    s, m = replicas.aggregate([1, 2], [3.0])
    assert list(s) == [1, 2] and list(m) == [3.0]


# ----------------------------------------------------------------- gloo ranks
def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _replica_run(doc, share):
    eng = Engine(scenario_from_dict(copy.deepcopy(doc), "replica"))
    rep = eng.run(specs=share)
    return eng, rep


def _rank_main(rank, world, port, doc, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        specs = build_requests(scenario_from_dict(copy.deepcopy(doc), "g").workload,
                               doc["horizon_s"])
        share = replicas.route(specs, world)[rank]
        eng, _ = _replica_run(doc, share)
        cores = replicas.core_set(rank, world, [-1] * world, list(range(4 * world)))
        tot, mx = replicas.aggregate([eng.counters["tokens_total"], eng.counters["merges"],
                                      len(share)], [eng.now, float(rank)], dist)
        gathered = [None] * world
        dist.all_gather_object(gathered, {"cores": cores, "ids": [s.id for s in share],
                                          "tokens": eng.counters["tokens_total"]})
        if rank == 0:
            out.put({"tot": tot.tolist(), "mx": mx.tolist(), "ranks": gathered})
    finally:
        dist.destroy_process_group()


def test_two_replicas_over_gloo_match_independent_runs():
    doc = make_doc(horizon_s=6)
    doc["workload"]["ls"]["rate"] = 3.0
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, doc, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    specs = build_requests(scenario_from_dict(copy.deepcopy(doc), "g").workload, doc["horizon_s"])
    shares = replicas.route(specs, world)
    solo = [_replica_run(doc, sh)[0] for sh in shares]
    # the reduction is the sum / max of what each replica computes alone
    assert res["tot"][0] == sum(e.counters["tokens_total"] for e in solo)
    assert res["tot"][1] == sum(e.counters["merges"] for e in solo)
    assert res["tot"][2] == len(specs)
    assert res["mx"][1] == world - 1
    for r in range(world):
        assert res["ranks"][r]["ids"] == [s.id for s in shares[r]]
        assert res["ranks"][r]["tokens"] == solo[r].counters["tokens_total"]
    assert not set(res["ranks"][0]["cores"]) & set(res["ranks"][1]["cores"])


@pytest.mark.gpu
def test_replica_cpu_pool_is_pinned(cuda):
    """A context created with a core set pins its CPU-attention workers to it
    (Cpus_allowed_list of each new thread is one core of the set)."""
    from paper_2603_12831_b200.models import get_transformer
    from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig

    allowed = sorted(os.sched_getaffinity(0))
    cores = allowed[:2]

    def threads():
        out = {}
        for tid in os.listdir("/proc/self/task"):
            try:
                txt = open(f"/proc/self/task/{tid}/status").read()
            except OSError:
                continue
            line = [x for x in txt.splitlines() if x.startswith("Cpus_allowed_list")][0]
            out[tid] = line.split(":")[1].strip()
        return out

    before = set(threads())
    ctx = HsContext(get_transformer("tiny"),
                    RuntimeConfig(max_rows=64, max_slots=8, kv_pages=64, max_pages_per_req=16,
                                  max_pos=1024, max_chunks=256, cpu_threads=3,
                                  host_kv_bytes=1 << 20, cpu_list=tuple(cores)))
    try:
        new = {t: a for t, a in threads().items() if t not in before}
        pinned = [a for a in new.values() if a in {str(c) for c in cores}]
        assert len(pinned) >= 2, new  # the ThreadPool's cpu_threads - 1 workers
        # the caller's own affinity is restored after the NUMA-local allocations
        assert sorted(os.sched_getaffinity(0)) == allowed
    finally:
        ctx.close()
