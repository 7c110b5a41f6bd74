"""Test infrastructure only: CPU restatement of the reference hot path (see gtopk_oracle.py)."""
