import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import torch, bench
from paper_1805_01208_b200 import KMeansSettings
from paper_1805_01208_b200.kmeans import partition_device
dev = torch.device("cuda")
c, pts_d, w_d, _ = bench.device_workload("C5", dev)
s = KMeansSettings(k=c["k"], epsilon=c["epsilon"], seed=0)
partition_device(pts_d, w_d, s, device=dev); torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
partition_device(pts_d, w_d, s, device=dev); torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(30)
