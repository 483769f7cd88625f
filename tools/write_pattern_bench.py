"""HBM write-pattern microbenchmark (B200): contiguous vs 128-byte row segments,
the pattern of the FWD2 / dX partial-output TMA stores (64-column boxes of a
[rows, 4096] bf16 matrix)."""
import torch

rows, d = 720896, 4096
buf = torch.empty(rows, d, dtype=torch.bfloat16, device="cuda")
nbytes = buf.numel() * 2


def timeit(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


t = timeit(lambda: buf.fill_(1.0))
print(f"contiguous fill: {t:.3f} ms, {nbytes / t / 1e6:.0f} GB/s")
cols = [buf[:, c:c + 64] for c in range(0, d, 64)]
t = timeit(lambda: [v.fill_(1.0) for v in cols])
print(f"64-column blocks (128 B per row): {t:.3f} ms, {nbytes / t / 1e6:.0f} GB/s")
cols = [buf[:, c:c + 256] for c in range(0, d, 256)]
t = timeit(lambda: [v.fill_(1.0) for v in cols])
print(f"256-column blocks (512 B per row): {t:.3f} ms, {nbytes / t / 1e6:.0f} GB/s")
src = torch.empty_like(buf)
t = timeit(lambda: src.copy_(buf))
print(f"copy (read + write): {t:.3f} ms, {2 * nbytes / t / 1e6:.0f} GB/s")
