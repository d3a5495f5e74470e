"""B200-native D2Q37 thermal Lattice Boltzmann hot path (arXiv 1703.00186).

The product is the C-ABI CUDA library ``liblb_d2q37.so`` (include/lb.h,
sources in ``csrc/``); ``lb`` is its thin Python binding.
"""
from .lb import (BC, MODE, COLLISION, Q, HALO, LBError, Lattice, constants, kwall, make_params,  # noqa: F401
                 nccl_unique_id, query_layout, exchange_plan, t0, tb_strip_height, lib, SO_PATH, EXPORTS)
