"""TEST INFRASTRUCTURE ONLY -- parity checkers for the CUDA path.

Two checkers live here:

* ``liboracle.so`` (``dpmrf_oracle.c``): a plain-C restatement of the
  reference's optimization hot path, citing proj/ file:line per function.
* ``_ref/libdpmrf_ref.so``: the reference library itself, compiled from its
  own sources by ``oracle/Makefile`` (present wherever it was built; it is
  git-ignored but travels to the GPU box with the snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.
"""
from .oracle import *  # noqa: F401,F403
