"""Context only (not part of the product): torch.sort (CUB radix sort on the GPU) on the
same inputs, L2 flushed, median of 5.  python tools/context_torch_sort.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402

l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(2 * l2, dtype=torch.uint8, device="cuda")
for name in ["c1", "c2", "c3", "c4", "c5f", "c5u"]:
    x = torch.from_numpy(synth.config(name)).cuda()
    if x.dtype == torch.uint64:
        x = x.view(torch.int64) ^ (-(2 ** 63))   # same order as u64
    torch.sort(x)
    ts = []
    for _ in range(5):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.sort(x, stable=False)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{name}: torch.sort {ts[2]:.3f} ms  ({x.numel() / ts[2] / 1e6:.2f} Gkeys/s, values+indices)")
    del x
    torch.cuda.empty_cache()
