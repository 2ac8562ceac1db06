"""Time the compiled reference (oracle/_ref) at 256^3: session setup and GN
matvecs at the bench linearisation (v = 0.5 v_syn, vt = -g)."""
import json, os, sys, time
sys.path.insert(0, ".")
from oracle import ref  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
t = time.time(); m0, v, m1 = ref.syn(n); t_syn = time.time() - t
t = time.time(); s = ref.Session(m0, m1, 0.5 * v, 1e-3, ref.Config(continuation=False, beta_target=1e-3)); t_sess = time.time() - t
g = s.gradient()
ts = []
for _ in range(2):
    t = time.time(); H = s.matvec(-g); ts.append(time.time() - t)
print(json.dumps(dict(n=n, syn_s=t_syn, session_s=t_sess, matvec_s=ts, timers=s.timers(), cores=os.cpu_count())))
