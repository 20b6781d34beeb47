"""CPU parity oracle for the emtrace propagation hot path.

TEST INFRASTRUCTURE ONLY.  This package restates the reference algorithm
(/root/reference/pkg/src/emtrace) on the CPU so that the CUDA product in
``paper_2303_11103_b200`` can be checked against it.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the
reported CPU baseline: the product never routes through it.

Pinning: ``tests/test_oracle_golden.py`` checks this oracle against golden
vectors produced by running the reference itself in the build container
(``tests/golden/make_golden.py``).
"""

from .port import *  # noqa: F401,F403
