"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

This package holds NONE of the method's arithmetic (no attention, no allocator,
no statistics, no batch-size rule).  It only produces inputs:

* ``hashgen`` -- a counter-based generator mapping logical coordinates
  (kind, request, position, layer, head, dim) to values k/128 in [-1, 1),
  exact in fp16 and bf16.  The CUDA library implements the same generator on
  the device (``paper_2503_05248_b200/csrc/device_common.cuh`` ``synth_key`` /
  ``synth_vals``, launched from ``csrc/kernels.cu``) so 150 GB of KV can be filled at HBM
  speed; ``tests/test_gpu_parity.py::test_device_generator_matches_host_generator`` checks
  the two bit-for-bit, ``tests/test_oracle_engine.py::test_hashgen_*`` pin the host side.
* ``trace`` -- request traces (arrival time, prompt length l_in, output length
  l_out) shaped like the paper's workloads, CSV I/O in the
  ``arrival_ms,l_in,l_out`` format of SPEC.md:100.
* ``configs`` -- the BASELINE.json configurations as concrete dictionaries.
"""
