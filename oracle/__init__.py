"""CPU oracle of the LS-CAT hot path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import anything under oracle/.  The product package (paper_2103_14409_b200) never does, and
the oracle never imports the product package: they share no code.

  oracle.table    - table analysis (argmin, ratios, bins, sums, percentiles), plain C via ctypes
  oracle.kernels  - fp64 numpy definitions of the suite kernels' outputs
"""
