# Is the step kernel's speed data-dependent? Same work, different physics:
# (a) default cavity, (b) t_hot = t_cold = t_inf (no driving: stays quiescent),
# (c) default cavity after 2000 iterations of spin-up.
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
from paper_2006_02602_b200 import capi
def timed(fl, pre=0, label=""):
    b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1), fluid=fl)
    b.initialize()
    b.run(3 + pre)
    tot, step = b.bench(300)
    print(f"{label:28s} step kernel {step:.4f} ms  -> {16777216 / step / 1e3:.0f} MCUPS", flush=True)
    b.close()
fl = capi.fluid_for_rayleigh(1e5)
timed(fl, 0, "default (from IC)")
flq = capi.fluid_for_rayleigh(1e5)
flq.t_hot = flq.t_inf
flq.t_cold = flq.t_inf
timed(flq, 0, "no driving (quiescent)")
timed(fl, 2000, "default after 2000 its")
