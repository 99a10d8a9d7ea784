"""CPU oracle (test/bench infrastructure only; never imported by the product path)."""
