"""SSS oracle — TEST INFRASTRUCTURE ONLY.

Plain fp64 CPU reference (``oracle/sss_oracle.cpp``) plus its ctypes wrapper.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2503_10148_b200`` never imports it.
"""
