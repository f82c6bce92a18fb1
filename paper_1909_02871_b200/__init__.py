"""B200-native (sm_100a) GF(2^w) region multiply-add and RLNC encoder: the hot
path of arXiv 1909.02871 behind a C ABI (include/gfrlnc.h).

    from paper_1909_02871_b200 import gf
    gf.init(256)
    B = gf.encode_batch(256, A, C)      # B[g,k,m] = sum_i C[g,i,k] * A[g,i,m]

The binding lives in `gf`; importing it loads libgfrlnc.so and fails loudly
when the library has not been built (there is no CPU fallback).
"""
import importlib

__all__ = ["gf"]


def __getattr__(name):
    if name == "gf":
        return importlib.import_module(__name__ + ".gf")
    raise AttributeError(name)
