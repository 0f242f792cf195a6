"""Ceiling check for K4: how fast does a generic gather of 15% of 256-byte rows run on this
GPU (torch index_select, same bytes as the C2 compaction), vs a plain copy of the same bytes."""
import torch

rows, d = 32 * 8 * 32768, 128
src = torch.randn(rows, d, device="cuda").to(torch.bfloat16)
keep = torch.rand(rows, device="cuda") < 0.15
idx = torch.nonzero(keep).squeeze(1)
out = torch.empty(idx.numel(), d, device="cuda", dtype=torch.bfloat16)
dense = torch.empty_like(out)


def t(fn, n=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


moved = 2 * idx.numel() * d * 2
ms_g = t(lambda: torch.index_select(src, 0, idx, out=out))
ms_c = t(lambda: dense.copy_(src[: idx.numel()]))
print(f"index_select 15% rows: {ms_g:.4f} ms  {moved / ms_g / 1e6:.0f} GB/s (read+write);  contiguous copy same bytes: {ms_c:.4f} ms  {moved / ms_c / 1e6:.0f} GB/s")
