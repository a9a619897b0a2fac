"""ORACLE package — test infrastructure only (see oracle/jacobi.py header).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import it.  It shares no code with paper_1901_07275_b200/.
"""
from .jacobi import (forward, inverse, forward_at, inverse_at, forward_axes, phi, gauss_jacobi,
                     p_all, recurrence_coefficients, mu0, kron_matrix, cauchy_h0, modified_q_all, phi_points,
                     phi_q_uniform, axis_matrix, forward_ex, adjoint_ex)

__all__ = ["forward", "inverse", "forward_at", "inverse_at", "forward_axes", "phi", "gauss_jacobi",
           "p_all", "recurrence_coefficients", "mu0", "kron_matrix", "cauchy_h0", "modified_q_all", "phi_points",
           "phi_q_uniform", "axis_matrix", "forward_ex", "adjoint_ex"]
