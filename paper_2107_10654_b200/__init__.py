"""B200-native sketched Tucker-ALS hot path (arXiv 2107.10654), drop-in for rtucker.h.

The product is the C-ABI shared library lib/librtucker_b200.so (hand-written
sm_100a CUDA + C++ host code); `rtucker` is its Python mirror (ctypes).
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "librtucker_b200.so")
