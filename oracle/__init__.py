"""CPU oracle for the O-SAM FOM/OpInf coupled time loop (arXiv 2511.20687).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_2511_20687_b200`) never imports it and shares no code
with it; the only common module is `osam_inputs` (seeded inputs, no method
arithmetic).

Plain, slow, obviously-correct NumPy/fp64 implementation of what the paper defines:
  fem.py       hex8 FE semi-discretisation, lumped mass, explicit Newmark (A.1)
  transfer.py  pointwise (trilinear) Schwarz projection Pi
  schwarz.py   FOM / OpInf-ROM subdomain models and Algorithm 1 controller
  opinf.py     POD, energy criterion, boundary POD and ridge OpInf
  exact.py     d'Alembert solution of the nu=0 bar (reading R28)

Parity status per function is in DESIGN.md ("Oracle pins"). Functions whose end-to-end
outputs have no closed form (ROM configs, c3/c4 runs) are "parity unpinned" end to end;
their components are pinned individually.
"""
