"""CPU oracle of the reference's hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker or the CPU baseline.  The product path
(``paper_1711_02473_b200``) never imports it and has no CPU fallback.

Contents
  sumfact_oracle.c   C restatement of the reference's per-cell kernels
                     (sum-factorised, OpenMP cell loop), see its header.
  cpu.py             ctypes driver of liboracle.so (built with gcc).
  dense.py           numpy restatement of the *unoptimised* lowering (dense
                     tabulation per point, no sum factorisation) — an
                     independent second oracle for small batches.
  gen_ref.py         builds oracle/_ref/: the reference's OWN emitted C
                     (scheduling.emit_c) for every BASELINE config, compiled
                     with an OpenMP cell-loop driver into shared libraries;
                     needs /root/reference at build time only.
  refc.py            ctypes driver of oracle/_ref (the "reference" CPU arm).

Pinning: tests/test_oracle.py checks cpu.py and dense.py against the golden
fixtures tests/golden/*.npz, which were produced by the reference itself
(tests/golden/make_golden.py, reference forms.evaluate_kernel).
"""
