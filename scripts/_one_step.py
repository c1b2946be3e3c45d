import sys; sys.path.insert(0, '/root/repo')
import numpy as np, synth, paper_1306_4080_b200 as pk
prob = synth.tiny(1, 40, 16, density=0.3, loss=0, c=3.0, P=5)
s = pk.Solver(prob)
r = s.step(np.arange(5, dtype=np.int32))
print(r['q'], r['n_touched'])
