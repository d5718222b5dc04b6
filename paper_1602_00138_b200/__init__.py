"""B200-native recycled-Krylov global-basis builder (arXiv 1602.00138 hot path).

Submodules:
  problem  -- host-side synthetic inputs (NormalStream, layouts, level sets, configs)
  romdot   -- Python mirror of the reference API over the C ABI (libromdot_b200.so)
  build    -- nvcc build of the in-tree library for sm_100a
"""
from . import problem  # noqa: F401
