"""B200-native exact-gradient evaluation for 3D density-based topology optimisation (arXiv 2104.12282).

The CUDA path lives in ``csrc/`` (built into ``lib/libtomo.so``) and is reached through
``paper_2104_12282_b200.tomo`` (ctypes binding of the C ABI in ``include/tomo.h``).
"""
