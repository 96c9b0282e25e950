"""CPU oracle for the DP-LLM decode hot path.

TEST INFRASTRUCTURE ONLY. Nothing in ``paper_2508_06041_b200`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may use it, and only as the
checker or as the timed CPU baseline, never as the product path.

``dpq_oracle`` is a numpy restatement of the reference ``dpq`` package's hot
path (``/root/reference/pkg/src/dpq``); every function cites the reference
file:line it follows. It is pinned against golden vectors produced by the
unmodified reference (``tests/golden/``, generator ``tools/make_golden.py``).
"""

from . import dpq_oracle  # noqa: F401
