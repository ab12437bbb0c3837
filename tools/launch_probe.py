"""Measurement tool (not product): event-timed launch cost of an empty 148-CTA kernel,
and of the small-batch kernels, after the bench's L2 flush (write 2x L2, read 2x L2),
by dynamic shared memory size.  Prints one JSON line per case."""
import ctypes
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "liblaunch_probe.so"))
    dev = torch.device("cuda:0")
    st = torch.cuda.current_stream()
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fw = torch.empty(int(2 * l2) // 4, device=dev)
    fr = torch.ones(int(2 * l2) // 4, device=dev)
    sink = torch.empty((), device=dev)

    def flush(i):
        fw.fill_(float(i))
        torch.sum(fr, dim=0, out=sink)

    def timed(fn, flushed, reps=200):
        for i in range(20):
            if flushed:
                flush(i)
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for i in range(reps):
            if flushed:
                flush(i)
            ev[i][0].record(st)
            fn()
            ev[i][1].record(st)
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        return ts[len(ts) // 2]

    for smem in (0, 48 * 1024, 200 * 1024, 225 * 1024):
        for flushed in (True, False):
            us = timed(lambda: lib.probe_launch(smem, 352, 148, ctypes.c_void_p(st.cuda_stream)), flushed)
            print(json.dumps({"case": "empty", "smem": smem, "flushed": flushed, "us": us}))
    # the library's small-batch kernel at cfg3, flushed and not
    import paper_2506_09282_b200 as hdc
    from hdc_inputs import CONFIGS, make_B, make_C, make_X
    for n in (1, 4, 16, 32):
        cfg = CONFIGS["cfg3_n%d" % n]
        X, B, C = (torch.from_numpy(a).to(dev) for a in (make_X(cfg), make_B(cfg), make_C(cfg)))
        m = hdc.Model(B, C, prec="fp32_tc")
        lab = torch.empty(n, dtype=torch.int32, device=dev)
        for flushed in (True, False):
            us = timed(lambda: m.infer(X, labels=lab), flushed)
            print(json.dumps({"case": "infer", "kernel": m.last_kernel(), "N": n, "flushed": flushed, "us": us}))
        m.close()


if __name__ == "__main__":
    main()
