"""CPU oracle for the InfoFlow-KV query-time context-assembly path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package, and only as the checker or the timed CPU baseline.  The product
package (``paper_2603_05353_b200``) never imports it.
"""

from .ifkv_oracle import *  # noqa: F401,F403
