"""CPU oracle (test infrastructure only; see moe_block.py header)."""
