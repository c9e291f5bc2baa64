"""CPU oracle for the blocked RQRCP / TRQRCP / TUXV hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1509_06820_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may use it, and only as the checker
or the timed CPU baseline, never as the product path.

``port`` is a numpy restatement of the reference algorithm
(/root/reference/pkg/src/rqrcp/{randomized,truncated,qrcp,kernels,rng}.py);
each function cites the reference file:line it follows.  It is pinned against
fixtures produced by running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.
"""

from . import port  # noqa: F401
