"""fp64 CPU oracle for Climber SUMI ranking inference (arXiv 2502.09888).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2502_09888_b200``) never imports it and the
two share no code; the only common module is ``synth`` (seeded inputs, no
arithmetic of the method).

Every function cites the PAPER.md passage it follows ("P:Lnnn" = PAPER.md line,
"S:Lnnn" = SPEC.md line, "G<n>" = reading n of SURVEY.md §8(c), restated in
DESIGN.md §2).

Parity status per function (DESIGN.md §2 lists the pins):
  extract, canonical_mask ............ pinned (brute force, closed forms)
  rmsnorm, softmax_tau, attention .... pinned (worked examples W1-W3, invariants)
  atl_* / encode_user / score_user ... pinned (torch-SDPA reduction, brute force,
                                       zero-weights closed form, rescaling invariants)
  bgf / head ......................... pinned (zero-weights closed form, N_b=1 case)
  bucket_pos, bucket_time, rel_bias .. pinned (boundary tables written independently,
                                       shift invariance, (W_q, f_b, tau) rescaling,
                                       torch-SDPA float-mask reduction, one-hot bias
                                       closed forms, SUMI == brute force with bias)
  absolute score values .............. parity unpinned (synthetic weights; the paper
                                       prints only AUCs)
"""
from .climber_oracle import *  # noqa: F401,F403
