import sys; sys.path.insert(0,'.')
import torch, paper_2205_03133_b200 as P
for cfg, n in ((0, 64), (3, 16)):
    P.synth_batch_gpu(cfg, n); torch.cuda.synchronize()
