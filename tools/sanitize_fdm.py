import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1506_05996_b200 as hx
from oracle import splitmix_vector
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
p = hx.Plan(hx.generate_cube_mesh(k), n)
r = splitmix_vector(p.N, 5)
print(np.linalg.norm(p.apply_fine(r)))
