"""Probe of the tensor cores' fp32 accumulation rounding (fp16 inputs, fp32 output) via
torch.mm(out_dtype=float32) (cuBLAS -> tcgen05 on sm_100): exact sum 1 + 0.75 ulp(1).
RN gives 1 + ulp, RZ (truncation) gives 1."""
import torch
ulp = 2.0 ** -23
for K in (16, 32, 64, 256):
    for sign in (1.0, -1.0):
        A = torch.zeros(128, K, dtype=torch.float16, device="cuda")
        B = torch.zeros(K, 128, dtype=torch.float16, device="cuda")
        A[:, 0] = sign
        B[0, :] = 1.0
        j = K - 1  # the small product in the last k position (another MMA k-block when K > 16)
        A[:, j] = 2.0 ** -12
        B[j, :] = sign * 3 * 2.0 ** -13
        C = torch.mm(A, B, out_dtype=torch.float32)
        v = C[0, 0].item()
        print(f"K={K:4d} sign={sign:+.0f}: result - sign = {(v - sign) / ulp:+.3f} ulp "
              f"(RN +-1, RZ 0)")
# many small terms: sum of 15 products of 0.3 ulp each on top of 1
A = torch.zeros(128, 16, dtype=torch.float16, device="cuda"); B = torch.zeros(16, 128, dtype=torch.float16, device="cuda")
A[:, 0] = 1.0; B[0, :] = 1.0
A[:, 1:] = 2.0 ** -12; B[1:, :] = 0.3 * 2.0 ** -11
C = torch.mm(A, B, out_dtype=torch.float32)
ex = 1.0 + 15 * (2.0 ** -12) * float(torch.tensor(0.3 * 2.0 ** -11, dtype=torch.float16))
print("15 small terms: got", (C[0, 0].item() - 1.0) / ulp, "ulp, exact", (ex - 1.0) / ulp, "ulp")
