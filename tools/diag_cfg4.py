import sys, numpy as np
sys.path[:0] = [".", "tests"]
import paper_2205_04295_b200 as pk
from oracle import rpie
from test_gpu_parity import rel_l2
geom = pk.Geometry.create(8.29e-10, 0.75, 20e-6, 512)
plan = pk.make_scan((3, 3), 64.0, 1.0, seed=4)
obj = pk.make_object(pk.canvas_shape_for(plan, 512), "spokes", seed=4)
for M in (5,):
    pw = (1.0,) if M == 1 else ((0.7, 0.3) if M == 2 else (0.6, 0.1, 0.1, 0.1, 0.1))
    probes = pk.make_probe(pk.ProbeSpec(M, pw, "disk", 120.0), geom)
    ds = pk.synthesize(obj, probes, plan, geom)
    for kap in (0, 10):
        cfg = pk.SolverConfig(alpha_obj=0.9, alpha_probe=0.9, beta=0.5, gamma=0.5, mode_count=M,
                              precision=sys.argv[1],
                              posref=pk.PosRefConfig(kappa=kap, warmup_iterations=0) if kap else None)
        st = pk.initialize(ds, cfg)
        ost = rpie.initialize(ds.patterns, ds.positions, 512, cfg)
        print("M", M, "kap", kap, "init", rel_l2(st.obj.cpu().numpy(), ost.obj),
              rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)))
        for it in range(2):
            pk.sweep(st, ds, cfg)
            rpie.sweep(ost, ds.patterns, 512, cfg)
            print("  it", it, rel_l2(st.obj.cpu().numpy(), ost.obj),
                  rel_l2(st.probe_stack.cpu().numpy(), np.stack(ost.probes)),
                  np.abs(st.positions.cpu().numpy() - ost.positions).max(),
                  st.error_trace[-1], ost.error_trace[-1], flush=True)
