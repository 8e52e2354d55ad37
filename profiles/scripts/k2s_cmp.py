import torch, sys
for N in sys.argv[1:]:
    a = torch.load(f"/tmp/k2_0_{N}.pt"); b = torch.load(f"/tmp/k2_1_{N}.pt")
    fa, fb = a.view(torch.float64), b.view(torch.float64)
    print("N", N, "bitwise:", bool(torch.equal(a, b)), "IEEE-equal:", bool(torch.equal(fa, fb)), "bit mismatches:", int((a != b).sum()))
