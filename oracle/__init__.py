"""Test infrastructure: CPU oracle (C restatement + reference driver)."""
