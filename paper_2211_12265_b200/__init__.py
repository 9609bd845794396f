"""B200-native batched CRYSTALS-Dilithium (round-3) engine -- Python binding over the
C ABI (include/dilithium_b200.h) of paper_2211_12265_b200/libdilithium_b200.so.

Only marshalling lives here.  There is no CPU fallback: if the CUDA library is missing
or no GPU is present, construction raises.
"""
from .engine import Engine, EngineError, LEVELS, lib_path, load_library  # noqa: F401
