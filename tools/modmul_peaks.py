import sys; sys.path.insert(0,'.')
import paper_1810_10121_b200 as P
ctx=P.Context(8192,[36,26,26,36],26,security=0)
for m in (0,1,2): print(m, ctx.modmul_peak(m)/1e12, "T modmul/s")
