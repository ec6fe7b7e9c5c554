"""ORACLE — test infrastructure only.

CPU restatements of the reference's fine-stage hot path, each citing the
reference file:line it follows.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
package, and only as the checker or as the timed CPU baseline — never on the
product path (paper_1512_06235_b200 never imports it).
"""
