import copy, sys, traceback
sys.path.insert(0, ".")
from oracle.scenarios import APPENDIX_B
from oracle.serve_oracle import device_weights, make_weights
from paper_2603_12831_b200 import tp
from paper_2603_12831_b200.engine import Engine
from paper_2603_12831_b200.models import TRANSFORMERS
from paper_2603_12831_b200.runtime import CudaStep, RuntimeConfig
from paper_2603_12831_b200.scenario import scenario_from_dict

cfg = TRANSFORMERS["tiny"]
dw = device_weights(make_weights(cfg, 0))
for world in (2,):
    rt = RuntimeConfig(max_rows=2048, max_slots=64, kv_pages=256, max_pages_per_req=16,
                       max_pos=2048, max_chunks=1024, cpu_threads=2, host_kv_bytes=64 << 20)
    ranks = [CudaStep(tp.shard_config(cfg, world), rt, weights=tp.shard_weights(dw, cfg, r, world))
             for r in range(world)]
    g = tp.TpStep(ranks)
    doc = copy.deepcopy(APPENDIX_B); doc["horizon_s"] = 1.6
    try:
        rep = Engine(scenario_from_dict(doc, "dbg"), step=g).run()
        print("world", world, "ok", rep.counters["tokens_total"])
    except Exception:
        traceback.print_exc()
        from paper_2603_12831_b200 import _lib
        print("last error:", _lib.last_error())
        for r, s in enumerate(ranks):
            print("rank", r, "logit_reqs", len(s._logit_reqs), "merge_L", len(s._merge_L), "iters", s.iterations)
