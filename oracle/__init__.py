"""CPU fp64 oracle — TEST INFRASTRUCTURE ONLY (tests/, smoke(), bench.py cpu_baseline).

The product path (paper_2601_03086_b200) never imports this package.
"""
