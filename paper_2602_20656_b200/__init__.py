"""lagom-b200: B200-native Lagom (arXiv 2602.20656).

Layers:
  * liblagom.so       drop-in C++ tuner API (include/lagom/*.hpp), bit-identical
                      to the reference's picks;
  * liblagom_coll.so  sm_100a collective kernels behind the C-ABI
                      include/lagom_coll.h (ring/tree AllReduce, ReduceScatter,
                      AllGather, AllToAll; SIMPLE / LL / LL128);
  * replay engine     the tuner's ProfileFn on real GPUs (lagom/b200.hpp).
Python modules here are thin bindings used by tests and bench.py.
"""
import os

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
__version__ = "0.1.0"
