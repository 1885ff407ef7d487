"""Device -> pinned host copy bandwidth: one stream vs several concurrent streams."""
import torch

n = 256 * 1024 * 1024  # 2 GiB of doubles
src = torch.empty(n, dtype=torch.float64, device="cuda").normal_()
dst = torch.empty(n, dtype=torch.float64).pin_memory()
for nstreams in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = n // nstreams
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                dst[k * chunk:(k + 1) * chunk].copy_(src[k * chunk:(k + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"streams={nstreams}: {n * 8 / ms / 1e6:.1f} GB/s ({ms:.1f} ms for 2 GiB)")
