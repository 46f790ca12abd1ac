import sys, faulthandler; sys.path.insert(0,'.')
faulthandler.dump_traceback_later(12, exit=False)
import numpy as np
from synth import planted_cliques
from paper_2210_16435_b200 import lib
g = planted_cliques(4, 6, 3, seed=7)
ctx = lib.sfairsc_build_operator(g.row_ptr, g.col, g.val, g.groups.astype(np.int32), 4, False, h=g.h)
print("built", ctx.info(), flush=True)
print("calling eigs", flush=True)
ev, X, st = lib.sfairsc_eigs(ctx, 4, 1e-10)
print(ev, st, flush=True)
