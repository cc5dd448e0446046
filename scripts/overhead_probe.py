"""Fixed costs of one launch (pfb_overhead_probe): empty kernel, + the NllArgs
parameter block, + constant-bank reads, + the accumulator epilogue."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1710_08826_b200 as pf
from paper_1710_08826_b200 import _lib as L
ctx = pf.device_context(0)
for mode, name in enumerate(["empty", "params_6KB", "const_reads", "finish_epilogue"]):
    out = ctypes.c_double()
    L.check(L.lib().pfb_overhead_probe(ctx.handle, mode, 21, ctypes.byref(out)), "probe")
    print(json.dumps({"mode": name, "us": out.value}), flush=True)
