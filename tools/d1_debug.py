"""Debug helper (GPU box): D1 of one recipe crop through the C ABI vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from synth import fields
import paper_2206_13932_b200 as dms
name = sys.argv[1]; shape = tuple(int(x) for x in sys.argv[2].split(","))
f = fields.make(name, shape=shape)
ref = oracle.run(f, nthreads=os.cpu_count(), want_pairs=False, want_d1=True)
rk = oracle.ranks(f)
d = dms.DMS(torch.from_numpy(f).cuda()); d.run_all()
print("nsig", len(ref.unpaired_top), "n0", len(ref.unpaired0))
try:
    d1 = d.diagram1()
    print("D1 equal", d1.tobytes() == ref.d1.tobytes())
    off, e = d.generators()
    print("gen equal", np.array_equal(off, ref.gen_off) and np.array_equal(e, ref.gen))
except dms.DMSError as ex:
    print("ERR", ex)
    import re
    m = re.search(r"sigma (\d+) tau ([0-9a-f]+) edge (-?\d+) owner (-?\d+)", str(ex))
    if m:
        sig, tau, j, o = int(m.group(1)), int(m.group(2), 16), int(m.group(3)), int(m.group(4))
        rh, rl = tau >> 32, tau & 0xffffffff
        inv = np.argsort(rk)
        print("sigma", sig, "tri", ref.unpaired_top[sig], "tau verts", inv[rh], inv[rl], "j", j)
        if j >= 0:
            print("un0[j]", ref.unpaired0[j], "oracle pair of that edge:", np.nonzero(ref.d1["birth_id"] == ref.unpaired0[j])[0])
        print("oracle pair of sigma", ref.d1[sig])
