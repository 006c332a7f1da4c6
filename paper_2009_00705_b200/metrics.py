"""Algorithmic byte / flop models of the hot-path kernels (DESIGN.md §"Roofline").

These count what the method must move, not what the kernels happen to move:
traffic above these numbers (ncu dram__bytes) is waste to remove.
"""


def schwarz_bytes_model(s, mesh=None, level=0) -> int:
    """One Schwarz sweep (eq 4.4): the packed symmetric inverses
    (8 B * n_k(n_k+1)/2 per subdomain), the subdomain index lists (4 B * n_k),
    and per node one read of r and W and a read-modify-write of u (32 B)."""
    i = s.info
    return int(8 * i["schwarz_packed"][level] + 4 * i["schwarz_nk_sum"][level] + 32 * i["level_n_dof"][level])


def apply_bytes_model(s, mesh=None, level=0) -> int:
    """One operator apply (eq 3.8): geometric factors (6 doubles per cubature
    point, Q = (p+1)^3), connectivity (4 B per element node), one read of u and
    one write of y per global node."""
    p = s.info["level_p"][level]
    Q = (p + 1) ** 3
    N = (p + 1) ** 2 * (p + 2) // 2
    E = s.info["n_elem"]
    return int(E * (48 * Q + 4 * N) + 16 * s.info["level_n_dof"][level])


def apply_flops_model(p: int, E: int) -> int:
    """Sum-factorised prism operator: 2 * (6 Qt Nt n1 + 6 Qt n1 Qv) + 15 Q per element."""
    n1 = p + 1
    nt = n1 * (n1 + 1) // 2
    qt = n1 * n1
    return int(E * (2 * (6 * qt * nt * n1 + 6 * qt * n1 * n1) + 15 * qt * n1))
