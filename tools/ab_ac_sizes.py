import os, sys, torch, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tools"))
import sweep
torch.cuda.set_device(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
out = []
for n in (512, 1024, 1536, 2048, 3072):
    r = sweep.cfg2(s, n=n, steps=10)
    out.append((n, round(r["integrate_steps_per_s"], 1)))
print(os.environ.get("TAG"), out)
