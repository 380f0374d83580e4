"""libopmm: B200 (sm_100a) hot path of the parallel Oculomotor Plant
Mathematical Model (arXiv 2007.09884) -- batched simulate + score + argmin
over candidate OPC vectors.  See include/opmm.h and DESIGN.md.

`from paper_2007_09884_b200 import opmm` gives the ctypes binding; it raises
ImportError if libopmm.so has not been built (there is no CPU fallback).
"""
__all__ = ["opmm"]
