"""Host->device bandwidth of one pinned 1352x1014x3 fp32 target (16.4 MB) on
this box: one copy, and the copy split over 2 / 4 streams (copy engines)."""
import torch

x = torch.empty(1014 * 1352 * 3, dtype=torch.float32).pin_memory()
y = torch.empty_like(x, device="cuda")
for parts in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(parts)]
    xs, ys = x.chunk(parts), y.chunk(parts)
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rep in range(23):
        if rep == 3:
            e0.record()
        for s, a, b in zip(streams, xs, ys):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                b.copy_(a, non_blocking=True)
        for s in streams:
            main.wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("h2d 16.4 MB in %d part(s): %.3f ms, %.1f GB/s" % (parts, ms, x.numel() * 4 / ms / 1e6))
