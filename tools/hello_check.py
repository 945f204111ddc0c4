import ctypes, torch, os
lib = ctypes.CDLL(os.path.join(os.path.dirname(__file__), "libhello.so"))
lib.hello_inc.argtypes = [ctypes.c_void_p, ctypes.c_long, ctypes.c_void_p]
x = torch.zeros(1000, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    rc = lib.hello_inc(x.data_ptr(), x.numel(), s.cuda_stream)
s.synchronize()
print("rc", rc, "sum", x.sum().item(), "torch cuda", torch.version.cuda, "nccl", torch.cuda.nccl.version())
