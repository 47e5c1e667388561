"""Print the cached .cu/.cubin of a workload's set module (for SASS /
ptxas inspection here, without a GPU): python tools/module_path.py case13659"""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2510_12897_b200 import _lib, jit  # noqa: E402
from paper_2510_12897_b200.device import host_layout  # noqa: E402
from paper_2510_12897_b200.workloads import build_workload  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "case13659"
gm = int(sys.argv[2]) if len(sys.argv) > 2 else None
plan = build_workload(name, lower_to_gpu=False).plan
src = host_layout(plan, gm).source
jit.compile_module(src)
key = hashlib.sha256((src + "\0" + " ".join(jit.NVRTC_OPTIONS) + "\0" + _lib.nvrtc_version()).encode()).hexdigest()
print(jit.CACHE_DIR / f"{key}.cubin")
