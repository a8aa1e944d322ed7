"""stgmg oracle — plain, slow, fp64 CPU implementation of the hot path of arXiv:2303.06742.

TEST INFRASTRUCTURE ONLY.  Nothing under ``oracle/`` is part of the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may
import or execute it.  The product path (``paper_2303_06742_b200``) never imports this package and
shares no code, header, table or constant generator with it; both sides only share the seeded input
generators of ``stgmg_inputs`` (which hold none of the method's arithmetic).

Every function cites the PAPER.md passage it follows as ``P:Ln`` (line of /root/reference/PAPER.md)
plus the LaTeX label of the equation / algorithm.  Where the paper is silent or garbled the reading
taken is the one listed in DESIGN.md §"Readings" (A1..A35, numbering of SURVEY.md §8(c)).

Modules
  basis      1D quadrature / Lagrange tables (Gauss, Gauss–Lobatto, right Gauss–Radau)
  temporal   dG(k) temporal constants T, omega_hat, chi_hat(-1), theta
  mesh       structured levels, DoF layout (Eq:DefXn)
  element    element matrices by tensor Gauss quadrature (Def:ACB, Def:ab)
  assembly   element slab matrices, global sparse A_n, element-by-element apply
  transfer   prolongation by interpolation, restriction = transpose
  vanka      vertex patches, A_P, equilibrated inverses, Algorithm 1
  mg         V-cycle
  lshape     3D L-shape benchmark: Q_r^d / P_{r-1}^disc, SIP B_gamma, directional BCs
  gmres      flexible GMRES(m), right preconditioned
  loads      load functionals, slab RHS, initial data, manufactured solutions
  errors     space-time error norms for the Tab:3 / Tab:App1 pins

Parity status per function is listed in DESIGN.md §"Oracle pins"; none is "parity unpinned"
except the GMRES iteration counts of the BASELINE configs (no printed counts exist).
"""
