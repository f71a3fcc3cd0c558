"""GPU diagnostics that check the device path against the oracle (test infrastructure: they
live under tests/ because only tests may call the oracle).  Run them as scripts, e.g.
``python tests/diagnostics/parity_report.py C2`` -- pytest does not collect them."""
