"""paper_2306_03622_b200 — B200-native swap-in-and-execute (FaaSwap, arXiv 2306.03622).

The product is libfsw.so (include/fsw.h): host store, weight pool, swap kernels and
flag-gated sm_100a layer kernels.  This package holds its sources (csrc/), the in-tree
build (build.py) and the ctypes binding (fsw.py).  It never imports the oracle.
"""
from .fsw import (  # noqa: F401
    Arena, FswError, Result, Runtime, lib, NO_OVERLAP, DMA_BASELINE, HOST_WC, HOST_ONLY,
    ORDER_EXEC, ORDER_REVERSE, ORDER_RANDOM, SWAP_RESIDENT, SWAP_HOST, ENGINE_AUTO, ENGINE_SM, ENGINE_DMA,
    NO_PEER_SWAP, SWAP_PEER, SWAP_STRIPED, Scheduler, ENGINE_SMZ, ENGINE_DMAZ, REG_LINK_CODE,
    DEBUG_POISON, FAULT_NONE, FAULT_DROP_PIECE, FAULT_DROP_GROUP, ENGINE_DMAZT,
)
