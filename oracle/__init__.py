"""fp64 CPU oracle for SparVAR's block-sparse cross-scale attention hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import this package.  The product path
(`paper_2602_04361_b200/`) never imports it and shares no code with it; the only thing the two
have in common is the seeded input generator in `synth/`, which holds none of the method's
arithmetic.

Every function is a plain, slow, literal transcription of a definition in the paper
(/root/reference/PAPER.md, cited as PAPER.md:<line> with the section/equation) in the order the
paper states it, in float64 (floating point) or exact integers / Fractions (geometry).  Where the
paper is silent or garbled, the reading taken is the one in SURVEY.md §8(c) and DESIGN.md
"Readings"; each such spot is marked `READING n`.

Modules
  geometry   O1/O2  scale schedule, prefix sums, global-index decomposition, blocks
  csla       O3     cross-scale local token mask, sink mask, block aggregation (Eq. block_mask)
  predictor  O4     decision-scale block mass, Top-K / threshold selection, sink union
  mapping    O5     query-block homography phi, Decompose-Align-Project (footprint / point)
  attention  O6-O8  merge to block lists, block-sparse attention, dense attention, brute force

Pins (what ties each function to something other than itself) are listed per module header and
tested under `tests/test_oracle_*.py` (all `-m "not gpu"`).  No function here is "parity
unpinned".
"""
