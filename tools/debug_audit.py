"""Debug: host-side recheck of the lazily relaxed bounds before every assign round."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden"))
import numpy as np
import cases
from oracle import geographer_oracle as O
from paper_1805_01208_b200 import KMeansSettings
from paper_1805_01208_b200 import kmeans as K

orig = K.DevicePartitioner._assign
state = {"round": 0}

def checked(self):
    k, d = self.settings.k, self.d
    ks = self.kstate.cpu().numpy()
    infl, S, T = ks[:k], ks[k:2*k], ks[2*k:]
    A = self.aargs
    a = self.A.cpu().numpy(); ub = self.UB.cpu().numpy(); lb = self.LB.cpu().numpy()
    X = self.X.cpu().numpy().T
    cen = self.centers_d.cpu().numpy()
    if A.list is None: idx = np.arange(A.m)
    else: idx = self.active_idx.cpu().numpy()[:A.m]
    pts = X[idx]
    mat = np.stack([O.effdist(pts, cen[c], infl[c]) for c in range(k)], axis=1)
    aa = a[idx]
    has = aa >= 0
    e = A.bound_err
    Sa, Ta = S[np.where(has, aa, 0)], T[np.where(has, aa, 0)]
    ube = np.where(has, Sa * ub[idx] + Ta + e * (np.abs(Sa * ub[idx]) + Ta), np.inf)
    lbe = np.maximum(A.lb_scale * lb[idx] - A.lb_shift - e * (A.lb_scale * lb[idx] + A.lb_shift), 0)
    own = mat[np.arange(len(idx)), np.where(has, aa, 0)]
    second = np.partition(mat, 1, axis=1)[:, 1] if k > 1 else np.full(len(idx), np.inf)
    v1 = has & (ube < own); v2 = lbe > second
    if v1.any() or v2.any():
        print(f"round {state['round']}: ub viol {v1.sum()} lb viol {v2.sum()} m={A.m} lbA={A.lb_scale} lbB={A.lb_shift}")
        for j in np.flatnonzero(v1 | v2)[:5]:
            print("  pos", idx[j], "a", aa[j], "ub~", ub[idx[j]], "ube", ube[j], "own", own[j], "lb~", lb[idx[j]], "lbe", lbe[j], "second", second[j], "argmin", mat[j].argmin())
    state["round"] += 1
    return orig(self)

K.DevicePartitioner._assign = checked
name = sys.argv[1] if len(sys.argv) > 1 else "u3_k64_audit"
spec = next(c for c in cases.PARTITION_CASES if c["name"] == name)
pts, w = cases.partition_inputs(spec)
s = dict(spec["settings"]); 
part, stats = K.balanced_kmeans_points(pts, w, KMeansSettings(**s), return_stats=True)
print("audit:", stats.audited_point_iterations, stats.bound_violations, stats.skip_check_failures)
