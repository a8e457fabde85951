"""Independent serving replicas, one per GPU.

The reference has no multi-GPU path: its cluster is one engine with
`gpu_count`/`tp_degree` folded into the latency models (engine.py:277-280,
latency.py:141-147).  OmniServe's paper runs each GPU with private queues and
an equal share of the host cores.  Here a replica is one
process per GPU (torch.distributed, one rank each) that owns its engine,
GPU KV, residual store, mailboxes and a CPU-attention pool pinned to cores of
the GPU's NUMA node.  There is no data-path collective: requests are
independent, so a replica never exchanges tensors with another.  The only
cross-rank traffic is the end-of-run reduction of the bench counters.

* `core_set`   - the replica's CPU cores: the NUMA node of its GPU, split
                 into equal blocks of whole physical cores among the GPUs on
                 that node (SMT siblings stay together).
* `route`      - a deterministic router splitting one global trace over the
                 replicas, round-robin per service class (the reference has
                 none; config 3's "8 independent replicas" can also use
                 per-replica seeds, `replica_seed`).
* `aggregate`  - sum of per-rank counters and max of per-rank times.
"""

from __future__ import annotations

import os
from pathlib import Path
from typing import Iterable, Optional, Sequence

import numpy as np

from .workload import RequestSpec, ServiceClass

_SYS = Path("/sys")


# ----------------------------------------------------------------- topology
def parse_cpulist(text: str) -> list[int]:
    """'0-3,8,10-11' -> [0, 1, 2, 3, 8, 10, 11] (the kernel's cpulist format)."""
    out: list[int] = []
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def gpu_pci_bus_id(device: int) -> Optional[str]:
    """PCI bus id ('0000:1b:00.0') of a CUDA device, or None without a GPU."""
    try:
        import torch

        if not torch.cuda.is_available():
            return None
        p = torch.cuda.get_device_properties(device)
        dom = getattr(p, "pci_domain_id", 0)
        return f"{dom:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    except Exception:
        return None


def gpu_numa_node(device: int, sysfs: Path = _SYS) -> int:
    """NUMA node of a GPU from sysfs (-1 when unknown)."""
    bus = gpu_pci_bus_id(device)
    if bus is None:
        return -1
    try:
        return int((sysfs / "bus/pci/devices" / bus.lower() / "numa_node").read_text())
    except (OSError, ValueError):
        return -1


def node_cpus(node: int, sysfs: Path = _SYS) -> list[int]:
    try:
        return parse_cpulist((sysfs / f"devices/system/node/node{node}/cpulist").read_text())
    except OSError:
        return []


def physical_cores(cpus: Iterable[int], sysfs: Path = _SYS) -> list[tuple[int, ...]]:
    """Group logical CPUs into physical cores (SMT siblings together), in
    order of each core's lowest CPU id."""
    cpus = sorted(set(cpus))
    allowed = set(cpus)
    seen: set[int] = set()
    cores: list[tuple[int, ...]] = []
    for c in cpus:
        if c in seen:
            continue
        try:
            sib = parse_cpulist(
                (sysfs / f"devices/system/cpu/cpu{c}/topology/thread_siblings_list").read_text())
        except OSError:
            sib = [c]
        group = tuple(s for s in sorted(sib) if s in allowed) or (c,)
        seen.update(group)
        cores.append(group)
    return cores


def core_set(local_rank: int, local_world: int, gpu_nodes: Optional[Sequence[int]] = None,
             allowed: Optional[Iterable[int]] = None, sysfs: Path = _SYS) -> list[int]:
    """The CPU-attention cores of replica `local_rank` among `local_world`
    GPU replicas on this host.

    GPUs on the same NUMA node share that node's allowed cores in equal,
    contiguous blocks of physical cores; GPUs whose node is unknown share all
    allowed cores the same way.  Blocks of different replicas are disjoint.
    """
    if not 0 <= local_rank < local_world:
        raise ValueError(f"local_rank {local_rank} outside [0, {local_world})")
    allowed = sorted(allowed if allowed is not None else os.sched_getaffinity(0))
    if gpu_nodes is None:
        gpu_nodes = [gpu_numa_node(i, sysfs) for i in range(local_world)]
    node = gpu_nodes[local_rank]
    pool = [c for c in node_cpus(node, sysfs) if c in set(allowed)] if node >= 0 else []
    peers = [r for r in range(local_world) if gpu_nodes[r] == node] if pool else \
        list(range(local_world))
    if not pool:
        pool = allowed
    cores = physical_cores(pool, sysfs)
    k = len(peers)
    i = peers.index(local_rank)
    per = len(cores) // k
    if per == 0:  # fewer cores than replicas: share round-robin
        mine = cores[i % len(cores):i % len(cores) + 1]
    else:
        mine = cores[i * per:(i + 1) * per]
    return sorted(c for core in mine for c in core)


# ----------------------------------------------------------------- routing
def route(specs: Sequence[RequestSpec], n: int) -> list[list[RequestSpec]]:
    """Split one arrival-ordered trace over `n` replicas: the k-th request of
    each service class goes to replica k mod n.  Deterministic, disjoint and
    covering; each replica's list stays in arrival order."""
    if n < 1:
        raise ValueError("need at least one replica")
    out: list[list[RequestSpec]] = [[] for _ in range(n)]
    seen = {ServiceClass.LS: 0, ServiceClass.BE: 0}
    for s in specs:
        out[seen[s.cls] % n].append(s)
        seen[s.cls] += 1
    return out


def replica_seed(seed: int, rank: int) -> int:
    """Per-replica workload seed for independently generated traces
    (config 3: 8 replicas with seeds 0..7)."""
    return seed + rank


# ----------------------------------------------------------------- reduction
def aggregate(sums: Sequence[float], maxes: Sequence[float], dist=None
              ) -> tuple[np.ndarray, np.ndarray]:
    """Whole-job totals: per-rank `sums` added, per-rank `maxes` maxed
    (device-timed windows: the job is as slow as its slowest replica)."""
    s = np.asarray(sums, dtype=np.float64)
    m = np.asarray(maxes, dtype=np.float64)
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return s, m
    import torch

    ts, tm = torch.from_numpy(s.copy()), torch.from_numpy(m.copy())
    dist.all_reduce(ts, op=dist.ReduceOp.SUM)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    return ts.numpy(), tm.numpy()


def mem_available_bytes() -> int:
    """MemAvailable of this host (/proc/meminfo); a large value if unknown."""
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 50
