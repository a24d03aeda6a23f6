"""CPU oracle for the Radar-STDA forward pass — TEST INFRASTRUCTURE ONLY.

Nothing under `oracle/` is product code.  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py`'s `cpu_baseline` / `--impl reference` leg may import it, and only as
the checker or the timed CPU baseline — never as the thing measured or shipped.
The product path (`paper_2307_09063_b200`) never imports this package.

Two independent restatements of `stda.StdaNet.forward` in eval mode
(reference `pkg/stda/src/stda/model.py:185-199`):

* `port`  — op-for-op restatement on torch CPU ops (conv2d / conv_transpose2d /
  batch_norm / relu / mean / conv1d / sigmoid), the exact arithmetic the reference
  dispatches to (oneDNN / ATen CPU).  This is the parity oracle and the CPU
  baseline ("kind": "port").
* `np64`  — a float64 numpy restatement built from the textbook definitions
  (im2col cross-correlation, scatter-form transposed convolution).  It shares no
  code with `port` and gives the fp64 noise floor.

Parity is PINNED: both restatements are checked against golden vectors produced
by running the real reference (`stda` imported from `/root/reference`) in the
build container — see `tests/golden/make_golden.py` and
`tests/test_oracle_golden.py`.
"""
