"""B200-native DeltaCNN engine (arXiv 2203.03996): Python binding of libdcnn.so.

Argument marshalling only -- every step of the frame-delta path runs in the
sm_100a kernels behind the C ABI declared in ``include/dcnn.h``.  There is no
CPU fallback: importing this package fails loudly when ``libdcnn.so`` is
missing (build it with ``python -m paper_2203_03996_b200.build``).
"""
from ._lib import (DeltaNet, DcnnError, load_library, OP_CODES, ACT_CODES,  # noqa: F401
                   BUF_DELTA, BUF_MASK, BUF_XA, BUF_XT, BUF_OUT, BUF_POOLA, LIB_PATH,
                   KCLASS_CONV, KCLASS_TILES, KCLASS_POINTWISE, KCLASS_INPUT,
                   FLAG_NO_TENSOR_CORES, FLAG_FP32_CACHES, FLAG_HYBRID_DISPATCH, FLAG_PER_PIXEL)
