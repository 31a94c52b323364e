"""Host->device copy bandwidth from pinned memory for the e2e leg's 128 MiB
per step: one stream vs. several streams / chunk sizes."""
import torch

dev = torch.device("cuda", 0)
N = 128 << 20
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device=dev)


def run(chunk, nstreams, reps=10):
    sts = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    main = torch.cuda.current_stream(dev)

    def once():
        ev = []
        for i, off in enumerate(range(0, N, chunk)):
            st = sts[i % nstreams]
            st.wait_stream(main)
            with torch.cuda.stream(st):
                d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
        for st in sts:
            main.wait_stream(st)
    once()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        once()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return round(N / ms / 1e6, 1)


for chunk in (N, 32 << 20, 8 << 20, 2 << 20):
    for ns in (1, 2, 4):
        print(f"chunk {chunk >> 20} MiB streams {ns}: {run(chunk, ns)} GB/s")
