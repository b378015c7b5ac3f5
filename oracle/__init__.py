"""CPU checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker (or
the timed CPU baseline); the product (paper_1806_07884_b200/) never does.
"""
