"""CPU oracle for the data-parallel mixed-precision LSTM training step of
arXiv 1912.00286.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The product path (``paper_1912_00286_b200``,
``libhdp.so``) never calls it and shares no code with it.

Plain, slow, obviously-correct NumPy in float64.  fp16 / fp32 rounding is
applied only at the pinned rounding points R0..R15 of SURVEY.md §8(c)
(listed again in DESIGN.md), because the paper fixes three precision
domains -- math, synchronisation, weight update --  but no
rounding points.

Modules
  binary16  the IEEE binary16 codec written from its definition
  schedule  learning-rate schedule, Eqs. 3-4 and the 0.1 clip
  lstm      LSTM forward / hinge loss (Eq. 6) / BPTT for one worker
  optim     averaging + SGD-momentum Eqs. 1-2 and Adam; the
            float32 emulation of the fused average+update kernel
  step      one synchronous data-parallel step over N simulated workers
            (steps 3-6)

Parity status: every function is pinned by
tests under tests/test_oracle_*.py against closed forms, the paper's /
SPEC's worked examples, finite differences, torch.nn.LSTM(float64) as an
independent library special case, and algebraic invariants.  The mixed-mode
*trajectory* (fp16 rounding interplay over many steps) has no exact value to
pin: "parity unpinned" for that aspect only -- it is compared to the GPU
within the north_star tolerance.
"""
