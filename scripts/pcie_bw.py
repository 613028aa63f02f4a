"""Host<->device copy bandwidth on this box (pinned memory): one copy vs the
same bytes split over several streams, each direction alone and both at once
(what tt_train_step_submit's uploads and downloads see)."""
import torch

N = 128 << 20  # bytes
h_up = torch.empty(N // 4, dtype=torch.float32).pin_memory()
h_dn = torch.empty(N // 4, dtype=torch.float32).pin_memory()
d_up = torch.empty(N // 4, dtype=torch.float32, device="cuda")
d_dn = torch.empty(N // 4, dtype=torch.float32, device="cuda")


def run(nstreams, up, down, reps=10):
    ss = [torch.cuda.Stream() for _ in range(2 * nstreams)]
    chunk = N // 4 // nstreams
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for i in range(nstreams):
            sl = slice(i * chunk, (i + 1) * chunk)
            if up:
                ss[i].wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(ss[i]):
                    d_up[sl].copy_(h_up[sl], non_blocking=True)
            if down:
                ss[nstreams + i].wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(ss[nstreams + i]):
                    h_dn[sl].copy_(d_dn[sl], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return N / (ms * 1e-3) / 1e9


for ns in (1, 2, 4):
    print(f"streams {ns}: H2D {run(ns, True, False):.1f} GB/s, D2H {run(ns, False, True):.1f} GB/s, "
          f"both {run(ns, True, True):.1f} GB/s per direction")
