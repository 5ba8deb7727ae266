import sys; sys.path.insert(0,'.')
import paper_1506_05996_b200 as hx
p = hx.Plan(hx.generate_cube_mesh(8), 4, coarse_sms=16)
print("coarse_sms", p.coarse_sms)
