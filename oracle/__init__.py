"""CPU oracle for the NSK training-step hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the timed
CPU baseline. The product path (paper_2409_11600_b200) never imports it.

* ref_ops.py   -- numpy restatement of the reference's own arithmetic
                  (pkg/src/nsk/tensor.py, autodiff.py, nn.py, builtins.py);
                  pinned against golden vectors produced by running the real
                  reference (tests/golden/gen_golden.py -> tests/golden/*.npz).
* restated.py  -- ops the reference does not have (conv2d, batchnorm, pooling,
                  im2col/col2im, crop/flip augmentation, embedding, GRU),
                  restated in float64 with the reference's conventions; pinned
                  by the reference's own finite-difference method
                  (gradcheck.py:89-138) and a torch-CPU float64 cross-check.
                  Parity of these ops is "pinned by FD", not by reference
                  outputs (the reference has no such ops).
* models.py    -- small CNN (C1) and CIFAR ResNet-18 (C2) training steps built
                  from the two modules above, parameter-for-parameter identical
                  to paper_2409_11600_b200.models (same names, seeds, order).
"""
