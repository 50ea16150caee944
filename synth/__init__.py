"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the DeltaCNN method (no convolution, no
delta propagation, no truncation).  It only produces:

* ``frames``  -- closed-form synthetic video: a static
  camera background plus hash-textured moving blobs, optional 1-LSB noise and a
  global flicker for the 100 %-update case, normalised with the ImageNet
  constants the paper names (§4).
* ``nets``    -- layer tables of the BASELINE.json configurations (single conv,
  the Fig. 2 toy network, HRNet-W32, YOLOv5s) with seeded random weights that
  are already BN-folded (§4).

Both the oracle (``oracle/``) and the product binding
(``paper_2203_03996_b200``) consume these objects; neither imports the other.
"""
