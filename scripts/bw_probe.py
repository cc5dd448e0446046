"""Read bandwidth of one pass over a device buffer: SIMT loads vs bulk-copy
rings (pfb_read_bw).  Calibrates what a streaming NLL kernel can reach.

    python scripts/bw_probe.py
"""

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1710_08826_b200 as pf
    from paper_1710_08826_b200 import _lib as L

    torch.cuda.set_device(0)
    ctx = pf.device_context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    for mb in (160, 640):
        buf = torch.ones(mb * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
        for mode, chunk in [(0, 1), (1, 16), (1, 32), (1, 64), (2, 8), (2, 16), (2, 32)]:
            out = ctypes.c_double()
            L.check(L.lib().pfb_read_bw(ctx.handle, ctypes.c_void_p(buf.data_ptr()), buf.numel() * 8, mode, chunk, 7,
                                        ctypes.byref(out)), "pfb_read_bw")
            print(json.dumps({"MB": mb, "mode": mode, "chunk_kb": chunk, "GBps": out.value}), flush=True)
        del buf


if __name__ == "__main__":
    main()
