"""Diagnostics: host->device copy bandwidth from pinned memory (the e2e bound of
hdc_model_infer_host) for one copy vs chunked copies on one or two streams."""
import torch


def timed(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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


def main():
    nbytes = 16384 * 617 * 4
    h = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    h.uniform_()
    d = torch.empty(nbytes // 4, dtype=torch.float32, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    cur = torch.cuda.current_stream()
    for nch in (1, 2, 4, 8, 16):
        for ns in (1, 2, 4):
            per = (h.numel() + nch - 1) // nch

            def go():
                for st in streams[:ns]:
                    st.wait_stream(cur)
                for i in range(nch):
                    st = streams[i % ns]
                    with torch.cuda.stream(st):
                        d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
                for st in streams[:ns]:
                    cur.wait_stream(st)
            ms = timed(go)
            print("H2D %.1f MB chunks=%2d streams=%d: %.3f ms  %.1f GB/s" % (nbytes / 1e6, nch, ns, ms, nbytes / ms / 1e6))
    hb = torch.empty(nbytes // 4, dtype=torch.float32).pin_memory()
    ms = timed(lambda: hb.copy_(d, non_blocking=True))
    print("D2H %.1f MB: %.3f ms  %.1f GB/s" % (nbytes / 1e6, ms, nbytes / ms / 1e6))

    def both():
        s0, s1 = streams[0], streams[1]
        s0.wait_stream(cur)
        s1.wait_stream(cur)
        with torch.cuda.stream(s0):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s1):
            hb.copy_(d, non_blocking=True)
        cur.wait_stream(s0)
        cur.wait_stream(s1)
    ms = timed(both)
    print("H2D+D2H concurrently %.1f MB each: %.3f ms" % (nbytes / 1e6, ms))


if __name__ == "__main__":
    main()
