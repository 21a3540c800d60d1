timeout 600 python tools/c3_block_diag.py C3 300 0 212 2>&1 | tail -20
