"""Host cost (us per call) of the torch CUDA primitives on the serving path."""
import time

import torch

dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
s1 = torch.cuda.Stream()
x = torch.empty(1 << 20, device=dev)


def t(name, fn, n=20000):
    for _ in range(200):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    print(f"{name:50s} {(time.perf_counter() - t0) / n * 1e6:7.2f} us")


t("torch.empty((1024,1024)) cuda", lambda: torch.empty((1024, 1024), device=dev))
t("torch.empty(1<<20, int64) cuda", lambda: torch.empty(1 << 20, dtype=torch.int64, device=dev))


def on_stream():
    prev = torch.cuda.current_stream(0)
    torch.cuda.set_stream(s1)
    try:
        return torch.empty((1024, 1024), device=dev)
    finally:
        torch.cuda.set_stream(prev)


t("empty via set_stream dance", on_stream)
t("x.record_stream(s1)", lambda: x.record_stream(s1))
t("torch.cuda.Event()", lambda: torch.cuda.Event())
e = torch.cuda.Event()
t("Event.record(s1)", lambda: e.record(s1))
t("s1.wait_event(e)", lambda: s1.wait_event(e))
t("torch.cuda.current_stream(0)", lambda: torch.cuda.current_stream(0))
t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("_cuda_getCurrentRawStream(0)", lambda: torch._C._cuda_getCurrentRawStream(0))
t("s1.cuda_stream", lambda: s1.cuda_stream)
t("x.data_ptr()", lambda: x.data_ptr())
t("x[:1000]", lambda: x[:1000])
t("x.numel()", lambda: x.numel())
t("torch.cuda.current_device()", lambda: torch.cuda.current_device())
cur = torch.cuda.current_stream(0)
t("cur.wait_stream(s1)", lambda: cur.wait_stream(s1))
