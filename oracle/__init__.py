"""CPU oracles -- TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke, bench.py cpu_baseline).

ckks_oracle.c / ckks.py / engine.py : RNS-CKKS residue oracle (the GPU must match it bit-for-bit)
sim.py                              : numpy restatement of the reference float64 simulator
"""
