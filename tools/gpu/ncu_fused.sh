python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
cat > /tmp/one.py <<'P'
import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2603_12831_b200.models import get_transformer
from paper_2603_12831_b200.runtime import HsContext, RuntimeConfig
ctx = HsContext(get_transformer("llama3-8b"), RuntimeConfig(max_rows=512, max_slots=8, kv_pages=64, max_pages_per_req=8, max_pos=128, max_chunks=64, cpu_threads=1, host_kv_bytes=0))
ctx.init_weights(0)
fn = ctx.lib.hs_probe_gemm
fn.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_float)]
us = C.c_float()
for f in (0, 1):
    print(fn(ctx.h, 3, 32, f, 1, C.byref(us)), us.value)
P
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_bf16 -o gpurun_out/prof_fused python /tmp/one.py > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/ncu_fused.log
