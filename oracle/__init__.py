"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Plain numpy/LAPACK reference of the paper's method (arxiv 2405.03584).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import it; the product package never does.

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` against
closed forms, brute-force enumeration, planted optima, assembled-system solves or
hand examples.  No function is "parity unpinned".
"""
