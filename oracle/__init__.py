"""DeltaCNN CPU oracle -- TEST INFRASTRUCTURE, not part of the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import anything under ``oracle/``.  The product
(``paper_2203_03996_b200``) never imports it and has no CPU fallback.

The oracle is plain numpy in fp64 (storage rounding to fp16/fp32 is emulated at
exactly the points where the method stores a value -- PAPER.md:388-389, §4.3 --
see DESIGN.md "Readings").  It shares no code with the CUDA path; the two meet
only through the seeded inputs of ``synth/``.

Parity pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function here
to something other than itself: the paper's worked examples (49-pixel dilation,
P:293-294; the ReLU counter-example; the 64-pixel window and the
12 544 / 589 824 / 14 745 600 cost example), closed forms
(Eq. 1 linearity, Eqs. 4-6 bookkeeping), torch's conv2d / max_pool2d in fp64 as
the textbook library routine, hand-computed fixtures under tests/golden/, and
brute force on tiny inputs.
"""
from .delta_oracle import (  # noqa: F401
    act_fn, conv2d, mask_conv, maxpool2d, avgpool2d, upsample_nearest, dilate_chebyshev,
    upsample_bilinear, mask_up_bilinear, conv_transpose2d, mask_conv_transpose,
    dense_forward, DeltaOracle, quantize, tile_window_counts, fold_bn,
)
