"""fp8b_peer_reduce_quantize on virtual peers (buffers of this one GPU): bytes
through HBM per second; the NVLink side cannot be measured on one GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_12334_b200 as F  # noqa: E402
from paper_1905_12334_b200.peer import PeerBuffer, reduce_quantize  # noqa: E402

F.init()
n = 1 << 26
for world in (1, 2, 4, 8):
    bufs = [PeerBuffer(4 * n) for _ in range(world)]
    for r, b in enumerate(bufs):
        F.fill_synthetic(b.view().view(torch.float32), "normal", r, 1.0)
    codes = torch.empty(n, dtype=torch.uint8, device="cuda")
    cnt = F.Counters()
    ptrs = [b.ptrs[0] for b in bufs]
    for _ in range(3):
        reduce_quantize(ptrs, 0, n, codes, counters=cnt)
    a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        reduce_quantize(ptrs, 0, n, codes, counters=cnt)
    b_.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b_) / 10
    print(f"world={world}  {ms * 1000:8.1f} us  {n * (4 * world + 1) / ms / 1e6:8.1f} GB/s")
    for bb in bufs:
        bb.close()
