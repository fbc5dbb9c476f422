"""B200-native particle hot path of the implicit-moment PIC cycle (arXiv 2507.20719).

  libpic.so      CUDA sm_100a kernels behind the C ABI of include/pic.h
  pic            ctypes binding with the C names (marshalling only)
  inputs         seeded synthetic workloads C1..C5 (shared with the tests' oracle)
  decomp         slab decomposition host logic (bounds, ownership, NCCL id broadcast)
"""
__version__ = "0.1.0"
