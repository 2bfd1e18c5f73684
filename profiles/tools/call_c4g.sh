set -x
mkdir -p gpurun_out
timeout 300 python tests/long_parity.py c4 c1 c2 c3 c5 --json gpurun_out/lp_diag.json > /dev/null 2>&1
python - <<'PY' > gpurun_out/c4_gamma_steps.txt 2>&1
import sys, numpy as np
sys.path[:0] = ['.', 'tests', 'oracle']
from paper_2507_04991_b200 import perrk as P, workloads as W
fx = np.load('tests/golden/long_c4.npz'); log = fx['log']
cfg = W.make_config('c4', steps=200)
semi = P.Semidiscretization(cfg.spec())
U0 = W.initial_state_for(cfg, (semi.node_x(), semi.node_y(), None))
semi.upload(U0)
rc = P.IntegratorConfig(tf=1e30, time=P.TimeControl(False, 0.0, P.CflRamp(cfg.cfl, cfg.cfl)), relaxation=cfg.relaxation)
_, _, _, recs = P.advance(semi, cfg.family, cfg.partition_map(), rc, 0.0, 200)
for k, r in enumerate(recs):
    print(k + 1, r.newton_iters, int(log[k, 3]), '%.17g %.17g %.3e %.6e %.6e' % (r.gamma, log[k, 2], r.gamma - log[k, 2], r.delta_h, log[k, 10]))
PY
echo done
