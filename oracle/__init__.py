"""CPU oracle for the MTraining hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import anything under oracle/.  The product path
(paper_2510_18830_b200/, libmtsa.so) never imports, links or executes it, and
this package never imports the product: the two share no code.  The only
shared module is synth/ (seeded random inputs, no method arithmetic).

Plain, slow, obviously-correct implementations, each function citing the
PAPER.md passage ("P:n" = line n of the paper text) it follows:

  vsidx.py        Alg. 1 index in the exact VS-IDX v1
                  arithmetic: fp32 round-to-nearest scores,
                  specified exp2, uint64 fixed-point reductions, integer top-p.
  _vsidx_ref.c    the same I1-I6 arithmetic in plain C (fast path for large S;
                  cross-checked bit-for-bit against vsidx.py on small inputs).
  sparseformat.py sparseformat and convert_index.
  attention.py    fp64 dense / sparse attention forward and backward
                  (Eq. 1, Eq. 12), merge_out_and_lse
                  (P:879).
  ring.py         flat and hierarchical sparse ring attention simulated over
                  logical ranks (Alg. 2).

Parity status of every function is listed in DESIGN.md §2.4 ("pins").
"""
