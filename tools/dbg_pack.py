import sys; sys.path.insert(0, '/root/repo')
import paper_1603_02526_b200 as fg
spec = fg.PackingSpec(300)
g = fg.build_packing(spec)
st = fg.init_state(g, seed=0)
fg.run(g, fg.RunConfig(max_iterations=3), state=st)
print("ok")
