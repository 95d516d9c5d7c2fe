"""CPU oracle for CoSine's batched verification step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2503_10325_b200``) never imports it and shares no code with it.

* ``cosine_oracle.c`` — plain fp64 C, every function citing the PAPER.md passage
  (or DESIGN.md reading) it follows.
* ``oracle.py`` — ctypes marshalling of numpy arrays into that C code.
* ``enum_check.py`` — exact rational (``fractions``) enumeration of the output
  distribution, the pin that the method reproduces the target distribution.

Parity pins: see DESIGN.md §4 ("what pins the oracle").  No oracle function is
"parity unpinned".
"""
from .oracle import *  # noqa: F401,F403
