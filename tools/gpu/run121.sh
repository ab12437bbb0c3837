for c in cfg3_n1 cfg3_n4 cfg3_n16 cfg3_n32; do timeout 300 python bench.py --config $c --prec fp32 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step']*1000,1), 'us', round(d['roofline']['kernel_ms']*1000,1), round(d['roofline']['frac'],3))"; done
cat > /tmp/sd.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
from hdc_inputs import CONFIGS, make_B, make_C
from hdc_inputs.device import make_X_device
import paper_2506_09282_b200 as hdc
cfg = CONFIGS["cfg3_n32"]; dev = torch.device("cuda:0")
X = make_X_device(cfg, dev, 0, 32)
m = hdc.Model(torch.from_numpy(make_B(cfg)).to(dev), torch.from_numpy(make_C(cfg)).to(dev), prec="fp32")
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
for n in (1, 32):
    for i in range(3):
        flush.fill_(float(i)); torch.cuda.synchronize()
        m.infer(X[:n], path="small"); torch.cuda.synchronize()
m.close()
PY
HDC_SMALL_DEBUG=1 timeout 120 python /tmp/sd.py 2>&1 | grep smallstream
