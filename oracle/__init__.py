"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the SpotServe mapping/migration path.

Nothing in the product package (`paper_2311_15566_b200`) may import this
package.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs use it, and only as the checker or
the timed CPU baseline -- never as the thing measured or shipped.

Contents
--------
* `port.py`          pure-Python restatement of the reference algorithm
                     (exact `Fraction` arithmetic, same loop structure and
                     float operation order as `spotsim`), each function citing
                     the reference file:line it follows.
* `spotkm_oracle.c`  plain-C restatement of the structured ("sweep") weight
                     builder, `_hungarian_max` and the two-step matcher, used
                     for full-size parity and as the multi-core CPU baseline.
* `cport.py`         ctypes loader for the compiled C oracle.

Parity pin: both restatements are checked against golden vectors produced by
running the real reference (`/root/reference/pkg/src/spotsim`) in the build
container -- see `tests/golden/gen_golden.py` and `tests/test_oracle_golden.py`.
"""
