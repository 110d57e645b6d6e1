"""CPU oracle for the Signal2SH -> LSC -> SH2Signal path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1808_01517_b200/`` imports this
package; only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may use it, and only as the checker or
as the timed CPU reference arm, never as the product path.

``port`` is a float64 numpy restatement of sphdwi 0.1.0 (the reference mounted
at /root/reference/pkg/src/sphdwi), function by function, with file:line
citations.  It is pinned against golden vectors produced by running the real
reference in the build container (``tests/golden/make_golden.py``).
"""

from . import port  # noqa: F401
