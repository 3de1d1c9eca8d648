"""Print the GEMM's one-wave cluster capacity (cudaOccupancyMaxActiveClusters) per (BN, cluster size)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2306_03622_b200 import Runtime, lib
with Runtime(gpu_ids=[0], pool_bytes=1 << 30):
    L = lib()
    f = L._ZN3fsw24gemm_max_active_clustersEii
    f.restype = ctypes.c_int
    for bn in (16, 32, 64, 128):
        print(bn, [(cz, f(bn, cz), f(bn, cz) * cz) for cz in range(2, 9)])
