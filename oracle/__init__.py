"""ORACLE — test infrastructure only.

CPU restatement of the reference hot path (arXiv 2209.08722 `skipm`,
/root/reference/pkg/src/skipm) used as the parity checker for the CUDA path.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import anything from this package; the product
package paper_2209_08722_b200 never does.

Pinned against the live reference by tests/golden/make_golden.py (run in the
build container where /root/reference exists) and tests/test_oracle_golden.py.
"""
