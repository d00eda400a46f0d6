"""B200-native (sm_100a) data-parallel hot path of NNTile (arXiv 2504.13236):
tiled GPT-2 block forward/backward + per-tile Adam behind the C ABI of
libnnt.so (include/nnt.h).

Submodules:
  nnt    ctypes binding with the ABI's names (argument marshalling only)
  model  BlockStack driver (torch for memory, streams, NCCL process groups)
  build  nvcc build of libnnt.so (sm_100a)
"""
import os as _os

LIB_PATH = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "libnnt.so")
