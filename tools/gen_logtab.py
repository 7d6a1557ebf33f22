"""Generate the 64-entry table of the matvec kernels' table-driven 0.5 log(x)
(paper_1705_05443_b200/csrc/kernels.cuh, g_logtab): entry j holds ic = fl(1 / c_j) and
lc = fl(-0.5 log ic) for c_j = 1 + (j + 0.5) / 64, computed with numpy longdouble (64-bit
mantissa on x86) and rounded to double.  lc belongs to the ROUNDED ic, so
0.5 log m = lc + 0.5 log1p(fma(m, ic, -1)) holds without a table bias."""
import numpy as np
ld = np.longdouble
print("__device__ const double2 g_logtab[64] = {")
for j in range(64):
    c = ld(1) + (ld(j) + ld(0.5)) / ld(64)
    ic = np.float64(ld(1) / c)
    lc = np.float64(-ld(0.5) * np.log(ld(ic)))
    print("    {%s, %s}," % (float(ic).hex(), float(lc).hex()))
print("};")

# exp table of exp_neg_tab: 2^(j/32) rounded to double, and the Cody-Waite split of ln2 / 32
import struct
ln2 = np.log(ld(2))
L = ln2 / ld(32)
b = struct.unpack("<Q", struct.pack("<d", float(np.float64(L))))[0] & ~((1 << 18) - 1)
hi = struct.unpack("<d", struct.pack("<Q", b))[0]
print("// ln2/32 = %s + %s, 32/ln2 = %r" % (float(hi).hex(), float(np.float64(L - ld(hi))).hex(),
                                              float(np.float64(ld(32) / ln2))))
print("static __device__ const double g_exptab[32] = {")
print("    " + ", ".join(float(np.float64(np.exp(ld(j) * ln2 / ld(32)))).hex() for j in range(32)))
print("};")
