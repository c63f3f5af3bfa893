"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no planning, no reduction,
no optimizer math).  It only produces:

* ``hashgen``   -- a counter-based generator (splitmix64) whose values are
                   exactly representable in bf16 and fp32, so the CPU oracle
                   and the GPU path see bit-identical inputs without a
                   transfer (SURVEY.md §8(d) "Inputs").
* ``workloads`` -- tensor shape lists and granularity *declarations* of the
                   BASELINE.json configs (model shapes are public configs;
                   granularity is the user's per-parameter declaration,
                   P:419 ``orig_param_policy``).  Resolving a declaration to
                   a block size g_t is method step a1 and lives on each side.
"""
