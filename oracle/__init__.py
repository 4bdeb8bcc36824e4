"""TEST INFRASTRUCTURE ONLY: fp64 CPU oracle of the AutoDeconJ light-field RL hot path.

Imported, called, linked or executed only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  It shares no code with paper_2208_11422_b200 (the CUDA product
path) and never imports it.  Pins: tests/test_oracle_*.py.

Parity unpinned (no independent pin exists in the reference):
  * the paper's "entropy maximum at the 7th iteration" (Fig. 2d) -- needs the C. elegans
    dataset and its wave-optics PSF (out of scope);
  * "entropy optimum ~ MSE optimum" -- found false on synthetic phantoms.
"""
