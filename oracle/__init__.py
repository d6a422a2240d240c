"""CPU ORACLE — test infrastructure only.

Nothing under ``oracle/`` is part of the product. Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it, and only as the checker (or as the timed
CPU restatement of the reference for the baseline arm). The product path in
``paper_2110_10762_b200`` never imports this package and fails loudly when its
CUDA library is missing.

Parity pinning: ``heat_oracle`` is checked against golden vectors produced by
the reference itself (``tests/golden/gen_golden.py`` imports ``pintlab`` from
``/root/reference/pkg/src`` in the build container and commits the outputs as
``tests/golden/*.npz``); see ``tests/test_oracle_golden.py``.
"""
