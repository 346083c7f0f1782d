"""TEST INFRASTRUCTURE ONLY -- the CPU oracle of the decompile path.

`oracle.port` restates the reference algorithm (unpyre.decompile_source,
/root/reference/pkg/src/unpyre/pipeline.py:143-160 and everything it calls) in
plain Python so parity can be checked, and the reference's CPU cost measured,
on machines where /root/reference does not exist (the GPU box).  It is pinned
against vectors produced by the real reference (tests/golden/*.jsonl and the
pool digests in tests/golden/pools.json): tests/test_oracle.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The product never does.
"""
