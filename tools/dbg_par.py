import os, sys, faulthandler
faulthandler.enable()
sys.path.insert(0, ".")
import osam_inputs as I
from paper_2511_20687_b200 import problem, osam
cfg = I.config("c1")
subs = problem.build(cfg)
problem.set_ics(cfg, subs)
print("built", flush=True)
rc, it = problem.run(cfg, subs, n_steps=2)
print("ran", rc, it.ravel(), flush=True)
