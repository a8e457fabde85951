"""Remote CPU hosts (the reference's hosts 1..cpu_hosts-1).

The reference's cluster has `cpu_hosts` CPU hosts; host 0 is the GPU's own
host (PCIe link), the others are remote (network link,
pkg/src/hybridserve/engine.py:329-331).  Offloaded BE requests go to the
local host while its memory lasts, then to the least loaded remote host
(`_distribute_offload`, engine.py:402-419), and their per-layer work items
are serviced on that host (engine.py:529-560).

A remote host here is a process running `hs_cpu_host_serve` (libhs,
csrc/cpu_remote.cpp): it owns the KV of the requests placed on it and runs
the same AVX-512/AMX host attention as the local pool.  A replica connects
to it with `HsContext.cpu_host_connect(host_id, addr, port)`; `CudaStep`
places a request's KV there when the engine offloaded it to that host.

    python -m paper_2603_12831_b200.cpu_host --model llama3-8b --port 0 --threads 16

prints `HS_CPU_HOST_READY port=<p>` once it listens.  `spawn()` starts one
on this machine (optionally pinned to a core set, e.g. the other NUMA
node), `RemoteHosts` starts `cpu_hosts - 1` of them for a scenario.
"""

from __future__ import annotations

import argparse
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path
from typing import Optional, Sequence

from . import _lib
from .errors import ConfigError
from .models import TransformerConfig, get_transformer

_ROOT = Path(__file__).resolve().parent.parent


def _model_cfg(m: TransformerConfig):
    from .runtime import HsModelCfg

    return HsModelCfg(m.d_model, m.n_layers, m.n_q, m.n_kv, m.head_dim, m.ffn, m.vocab,
                      m.rope_theta, m.norm_eps)


def model_args(m: TransformerConfig) -> list[str]:
    """Command-line form of a transformer geometry (for models built in code)."""
    return ["--dims", ",".join(str(x) for x in (m.d_model, m.n_layers, m.n_q, m.n_kv, m.head_dim,
                                                m.ffn, m.vocab, m.rope_theta, m.norm_eps))]


def serve(model: TransformerConfig, port: int = 0, bind: str = "127.0.0.1", threads: int = 4,
          max_slots: int = 1024) -> None:
    """Blocking: serves until a client asks for shutdown."""
    lib = _lib.load()
    mc = _model_cfg(model)
    _lib.check(lib.hs_cpu_host_serve(C.byref(mc), bind.encode(), port, threads, max_slots),
               "hs_cpu_host_serve")


class HostProcess:
    """One remote CPU host process on this machine."""

    def __init__(self, model: TransformerConfig, threads: int = 4, max_slots: int = 1024,
                 cpus: Optional[Sequence[int]] = None, bind: str = "127.0.0.1"):
        cmd = [sys.executable, "-m", "paper_2603_12831_b200.cpu_host", *model_args(model),
               "--threads", str(threads), "--max-slots", str(max_slots), "--bind", bind,
               "--port", "0"]
        env = dict(os.environ)
        env["PYTHONPATH"] = str(_ROOT) + os.pathsep + env.get("PYTHONPATH", "")
        preexec = (lambda: os.sched_setaffinity(0, list(cpus))) if cpus else None
        self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=None, env=env,
                                     cwd=str(_ROOT), preexec_fn=preexec, text=True)
        self.addr = bind
        self.port = -1
        line = self.proc.stdout.readline()  # blocks until the server listens (or exits)
        if not line.startswith("HS_CPU_HOST_READY"):
            self.proc.kill()
            raise ConfigError(f"remote CPU host failed to start: {line!r}")
        self.port = int(line.split("port=")[1])

    def stop(self, timeout_s: float = 10.0) -> None:
        if self.proc.poll() is None:
            try:
                shutdown(self.addr, self.port)
                self.proc.wait(timeout=timeout_s)
            except Exception:
                self.proc.kill()
                self.proc.wait()


def shutdown(addr: str, port: int) -> None:
    """Asks a remote host to exit (a BYE(1) message, csrc/cpu_remote.cpp)."""
    import socket
    import struct

    with socket.create_connection((addr, port), timeout=10) as s:
        s.sendall(struct.pack("<4i", 6, 0, 1, 0))


def spawn(model: TransformerConfig, **kw) -> HostProcess:
    return HostProcess(model, **kw)


class RemoteHosts:
    """The remote hosts 1..n of a scenario, started on this machine and
    connected to a replica's context (`attach`)."""

    def __init__(self, model: TransformerConfig, n: int, threads: int = 4,
                 max_slots: int = 1024, cpu_sets: Optional[Sequence[Sequence[int]]] = None):
        self.hosts = [HostProcess(model, threads=threads, max_slots=max_slots,
                                  cpus=cpu_sets[i] if cpu_sets else None) for i in range(n)]

    def attach(self, ctx) -> None:
        for i, h in enumerate(self.hosts, start=1):
            ctx.cpu_host_connect(i, h.addr, h.port)

    def close(self) -> None:
        for h in self.hosts:
            h.stop()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def main(argv: Optional[list[str]] = None) -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--model", default=None, help="transformer name (models.TRANSFORMERS)")
    ap.add_argument("--dims", default=None,
                    help="d,layers,n_q,n_kv,head_dim,ffn,vocab,rope_theta,norm_eps")
    ap.add_argument("--bind", default="127.0.0.1")
    ap.add_argument("--port", type=int, default=0)
    ap.add_argument("--threads", type=int, default=4)
    ap.add_argument("--max-slots", type=int, default=1024)
    a = ap.parse_args(argv)
    if a.dims:
        v = a.dims.split(",")
        m = TransformerConfig("remote", *[int(x) for x in v[:7]], rope_theta=float(v[7]),
                              norm_eps=float(v[8]))
    elif a.model:
        m = get_transformer(a.model)
    else:
        ap.error("--model or --dims is required")
    serve(m, a.port, a.bind, a.threads, a.max_slots)


if __name__ == "__main__":
    main()
