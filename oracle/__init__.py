"""UniAP CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the
CUDA product path (``paper_2307_16375_b200``); neither imports the other.

* ``oracle.oracle`` -- ctypes wrapper of the plain C oracle (``oracle.c``):
  builder' (the cost model), interval chain DP (Eq. 3 under
  Eq. 5), Pareto combine of Eq. 2, lexicographic traceback, Algorithm 1.
* ``oracle.brute`` -- pure-Python brute force over every stage-and-strategy
  assignment of tiny instances (Eqs. 2-8 evaluated literally).
"""
