"""Probe: does this box support NVLS multicast (driver attribute), and does
torch symmetric memory hand out a multicast address at world size 1?"""
import ctypes, os, socket
import torch
import torch.distributed as dist
libcuda = ctypes.CDLL("libcuda.so.1")
libcuda.cuInit(0)
dev = ctypes.c_int()
libcuda.cuDeviceGet(ctypes.byref(dev), 0)
val = ctypes.c_int(-1)
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = libcuda.cuDeviceGetAttribute(ctypes.byref(val), 132, dev)
print("cuDeviceGetAttribute(MULTICAST_SUPPORTED) rc", r, "value", val.value)
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as sm
try:
    print("backend", sm.get_backend(torch.device("cuda", 0)))
except Exception as e:
    print("get_backend", e)
buf = sm.empty(1024, dtype=torch.float32, device="cuda")
h = sm.rendezvous(buf, dist.group.WORLD.group_name)
print("multicast_ptr", getattr(h, "multicast_ptr", None), "buffer_ptrs", h.buffer_ptrs, "world", h.world_size)
print([a for a in dir(h) if not a.startswith("_")])
os.system("nvidia-smi -q | grep -i -A3 'fabric' | head -20; nvidia-smi topo -m | head -5")
dist.destroy_process_group()
