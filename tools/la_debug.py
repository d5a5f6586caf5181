import ctypes, os, sys
sys.path.insert(0, ".")
os.environ["HPS_B200_LIB"] = "abtest/ladbg/_hps_b200.so"
os.environ["HPS_GJ_LA"] = "1"
import torch
from paper_1612_02736_b200 import _ext
lib = _ext.load()
dbg = torch.zeros(8, dtype=torch.int32).pin_memory()
C = ctypes.CDLL("abtest/ladbg/_hps_b200.so")
C.hps_la_debug_buffer(ctypes.c_void_p(dbg.data_ptr()))
n, ncols, batch = 196, 256, int(sys.argv[1]) if len(sys.argv) > 1 else 148
g = torch.Generator(device="cuda").manual_seed(0)
A0 = torch.randn(batch, n, ncols, dtype=torch.float64, device="cuda", generator=g)
A0[:, :, :n] += n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda")
M = A0.clone()
piv = torch.empty(batch, n, dtype=torch.int32, device="cuda")
ws = torch.empty(int(lib.hps_gj_workspace_bytes(batch, n, ncols)), dtype=torch.uint8, device="cuda")
lib.hps_gj_invert_batched(batch, n, ncols, _ext.mat(M, n * ncols, ncols), piv.data_ptr(), ws.data_ptr(),
                          None, None, None, None, torch.cuda.current_stream().cuda_stream)
try:
    torch.cuda.synchronize()
    inv = torch.linalg.inv(A0[:, :, :n])
    print("ok, max err", (M[:, :, :n] - inv).abs().max().item() / inv.abs().max().item())
except Exception as e:
    print("FAILED", str(e)[:80])
print("dbg (code 1=empty 2=lab 3=full, k, parity, tid, block):", dbg.tolist())
h = (ctypes.c_longlong * 16)()
C.hps_la_prof(h)
names = {0: "P column loop", 1: "P wait empty", 2: "P publish", 3: "P wait la cols", 4: "P stage W (la)", 5: "P la tiles",
         6: "P load next", 8: "U wait full", 9: "U la chunk", 10: "U stage W", 11: "U tiles"}
items = (batch + 147) // 148
for i, nm in names.items():
    print(f"  {nm:16s} {h[i] / items:12.0f} cycles / matrix")

