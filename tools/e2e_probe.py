"""Diagnostics: where the end-to-end (host buffer) step time goes -- device-resident
inference time per chunk size, and hdc_model_infer_host under chunk-size overrides."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from hdc_inputs import CONFIGS, make_B, make_C          # noqa: E402
from hdc_inputs.device import make_X_device              # noqa: E402
import paper_2506_09282_b200 as hdc                      # noqa: E402


def timed(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts) // 2]


def gpu_only(fn, reps=20):
    """GPU time per call with the host enqueue hidden: the stream is held by a sleep
    kernel while the calls are queued behind it."""
    import time
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200_000_000)
    s.record()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    host = (time.perf_counter() - t0) / reps * 1e3
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps, host


def main():
    cfg = CONFIGS[os.environ.get("CFG", "cfg2")]
    prec = os.environ.get("PREC", "fp32_tc")
    dev = torch.device("cuda:0")
    X = make_X_device(cfg, dev, 0, cfg.N)
    B = torch.from_numpy(make_B(cfg)).to(dev)
    C = torch.from_numpy(make_C(cfg)).to(dev)
    m = hdc.Model(B, C, prec=prec)
    for n in (2048, 4096, 8192, 16384):
        if n > cfg.N:
            break
        ms = timed(lambda: m.infer(X[:n]))
        g, h = gpu_only(lambda: m.infer(X[:n]))
        print("device infer n=%6d: %.3f ms  (%.3f ms per 16384 rows); GPU-only %.3f ms, host enqueue %.3f ms"
              % (n, ms, ms * 16384 / n, g, h))
    Xh = X.cpu().pin_memory()
    yh = torch.empty(cfg.N, dtype=torch.int32).pin_memory()
    for rows in (2048, 4096, 8192, 16384):
        os.environ["HDC_HOST_CHUNK_ROWS"] = str(rows)
        ms = timed(lambda: m.infer_host(Xh, yh))

        def ten():
            for _ in range(10):
                m.infer_host(Xh, yh)
        ms10 = timed(ten, reps=3) / 10
        print("infer_host chunk=%6d: %.3f ms one call, %.3f ms per call back-to-back (%.2f M samples/s)"
              % (rows, ms, ms10, cfg.N / ms10 / 1e3))
    m.close()


if __name__ == "__main__" and not os.environ.get("BENCH_LIKE"):
    main()


def bench_like():
    """The bench.py e2e pattern: 2 warm-up calls, then 20 back-to-back calls, with
    per-call events on the compute stream."""
    cfg = CONFIGS[os.environ.get("CFG", "cfg2")]
    dev = torch.device("cuda:0")
    X = make_X_device(cfg, dev, 0, cfg.N)
    m = hdc.Model(torch.from_numpy(make_B(cfg)).to(dev), torch.from_numpy(make_C(cfg)).to(dev),
                  prec=os.environ.get("PREC", "fp32_tc"))
    for _ in range(3):
        m.infer(X)
    Xh = X.cpu().pin_memory()
    yh = torch.empty(cfg.N, dtype=torch.int32).pin_memory()
    for _ in range(2):
        m.infer_host(Xh, yh)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(21)]
    ev[0].record()
    for i in range(20):
        m.infer_host(Xh, yh)
        ev[i + 1].record()
    torch.cuda.synchronize()
    d = [ev[i].elapsed_time(ev[i + 1]) for i in range(20)]
    print("bench-like per call ms:", " ".join("%.3f" % x for x in d), " total %.3f" % ev[0].elapsed_time(ev[20]))
    m.close()


if __name__ == "__main__" and os.environ.get("BENCH_LIKE"):
    bench_like()
