"""Which call sites read device tensors back to pageable host memory during c2
outer steps (monkeypatched Tensor.cpu / item / tolist; development aid)."""
import collections, os, sys, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
sites = collections.Counter(); sizes = collections.Counter()
orig = {k: getattr(torch.Tensor, k) for k in ("cpu", "item", "tolist", "__float__", "__int__", "__bool__")}
active = [False]
def wrap(name):
    f = orig[name]
    def g(self, *a, **k):
        if active[0] and self.is_cuda:
            st = traceback.extract_stack(limit=4)[-2]
            key = f"{name} {os.path.basename(st.filename)}:{st.lineno} {st.line[:70]}"
            sites[key] += 1; sizes[key] += self.numel() * self.element_size()
        return f(self, *a, **k)
    return g
for k in orig:
    setattr(torch.Tensor, k, wrap(k))
sys.argv = [sys.argv[0]]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "prof_solve_timeline.py")).read()
src = src.split("run(2)")[0]
exec(compile(src, "prof_solve_timeline", "exec"))
run(2)
active[0] = True
run(4)
active[0] = False
for k, v in sites.most_common(30):
    print(f"{v:5d}  {sizes[k]:12d} B  {k}")
