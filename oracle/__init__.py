"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of the veScale-FSDP
RaggedShard/DBuffer collective step (arxiv 2602.22437), written from
/root/reference/PAPER.md (cited as P:<line>) and the readings of SURVEY.md
§8(c) (listed in DESIGN.md "Readings").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2602_22437_b200`` + ``librsdb.so``) never imports it, and this
package imports nothing from the product path; the only shared module is
``synth`` (seeded inputs and model shapes, no method arithmetic).

Modules
  planner  -- a1 granularity, a2 Alg. 1 planner (O1), validator, brute force,
              a3 per-rank segment / quantization-block tables
  dbuffer  -- a4/a5 AllGather + views, a6 grouped cast/scale, a7 ReduceScatter (O2, O3)
  adam8    -- a8 block-wise 8-bit Adam (O4; linear codes, or the dynamic map)
  codemap  -- N2 dynamic (tree) code map of the 8-bit states (R25)
  fp8      -- N2 FP8 E4M3 128x128 block quantization before the AllGather (R18-R20)
  muon     -- N3 distributed Muon, Algorithm 2 (R21-R24)

Parity status of every function is stated in its docstring; all are pinned
(tests/test_oracle_*.py) -- there is no "parity unpinned" function.
"""
