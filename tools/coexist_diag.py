"""Diagnostic: the worker service running beside bulk kernels, keys, engines
and the HBM store in one process (with TORCH_FIRST=1: torch initialised
before the service), under a 20 s faulthandler deadline."""
import faulthandler, sys, os, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
faulthandler.dump_traceback_later(20, exit=True)
import numpy as np, torch
import paper_2004_09252_b200 as pc
from paper_2004_09252_b200 import _native
from paper_2004_09252_b200.workers import WorkerPool, ClientId
from paper_2004_09252_b200.store import DevicePageStore
KEY = bytes(range(32))
if os.environ.get("TORCH_FIRST"):
    torch.zeros(1, device="cuda"); torch.cuda.synchronize(); print("torch initialised first", flush=True)
pool = WorkerPool(n_workers=4, keysource=lambda n: KEY)
def step(name, fn):
    t0 = time.time(); fn(); print(f"{name}: ok {time.time()-t0:.3f}s", flush=True)
step("key install", lambda: pc.DeviceKey.install(KEY, 0).destroy())
k = pc.DeviceKey.install(KEY, 0)
z = None
def mkz():
    global z; z = torch.zeros((64, 4096), dtype=torch.uint8, device="cuda")
step("torch zeros", mkz)
step("torch sync", lambda: torch.cuda.current_stream().synchronize())
step("device crypt", lambda: pc.crypt_pages(k, 0x1000, 1, z))
step("torch sync 2", lambda: torch.cuda.current_stream().synchronize())
def host_alloc_free():
    p = ctypes.c_void_p(); _native.call("pc_host_alloc", 1 << 20, ctypes.byref(p)); _native.call("pc_host_free", p)
step("pinned alloc/free", host_alloc_free)
eng = None
def mk(): 
    global eng; eng = pc.Engine(0, n_streams=2, chunk_pages=256)
step("engine create", mk)
step("host crypt pageable", lambda: pc.crypt_pages(k, 0x1000, 1, np.zeros((600, 4096), np.uint8), engine=eng))
step("engine destroy", lambda: eng.destroy())
st = None
def mks():
    global st; st = DevicePageStore(16, k)
step("store create", mks)
step("store evict/refault", lambda: (st.evict(ClientId(1, 0), 0x5000, bytes(4096)), st.refault(ClientId(1, 0), 0x5000)))
step("store close", lambda: st.close())
step("key destroy", lambda: k.destroy())
step("torch alloc", lambda: torch.empty(1 << 28, dtype=torch.uint8, device="cuda"))
step("empty_cache", lambda: torch.cuda.empty_cache())
pool.shutdown()
print("done")
