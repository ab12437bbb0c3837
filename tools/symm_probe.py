import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1)
torch.cuda.set_device(0)
from cuda.bindings import driver as cu
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
    a = getattr(cu.CUdevice_attribute, name)
    print(name, cu.cuDeviceGetAttribute(a, dev))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1024, dtype=torch.float32, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD)
    print("symm ok; multicast_ptr", h.multicast_ptr, "buffer_ptrs", h.buffer_ptrs, "signal_pad", h.signal_pad_ptrs)
    print([a for a in dir(h) if not a.startswith("_")])
except Exception as e:
    print("symm failed:", repr(e))
dist.destroy_process_group()
