"""CPU oracle for the SRHT sketch of RandomizedNNLS (arXiv 0812.4547).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_0812_4547_b200``) never imports it and shares
no code with it: the oracle has its own Philox, its own plan derivation, its own
(recursive) Walsh-Hadamard transform and its own NNLS solver.

Everything is plain float64 numpy, written to be checked against PAPER.md by eye:

* ``oracle.philox``  -- Philox4x64-10 (Salmon et al., SC'11), pure Python, plus the
  numpy library routine ``numpy.random.Philox`` used as a bulk generator.
* ``oracle.srht``    -- Algorithm 1 steps 1-4 and the sketch
  H~ D [A | b] of step 5, with the Hadamard-Walsh recursion of
  Section 2.
* ``oracle.nnls``    -- Definition 1 solved by the Lawson-Hanson
  active-set method the paper names, brute-force support
  enumeration, KKT certificate, and the Fig. 1 relative error.

Readings where the paper is silent or ambiguous are listed in DESIGN.md
("Readings", R1-R14); each function cites the one it uses.

Parity status: every function here is pinned by ``tests/test_oracle_*.py``
against values that do not come from the oracle itself (published Philox
known-answer vectors, scipy.linalg.hadamard, closed forms, brute force,
scipy.optimize.nnls).  The only unpinned quantity is Theorem 1's (1+eps) bound
itself, whose constant c_o is unspecified: "parity unpinned" for the
bound, see DESIGN.md.
"""

from . import philox, srht, nnls  # noqa: F401
