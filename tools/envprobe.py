import os, torch
torch.zeros(1).cuda()
print("ENV", sorted(k for k in os.environ if any(s in k.upper() for s in ("NV", "CUDA", "INJ", "PRELOAD", "NSIGHT", "NCU"))))
