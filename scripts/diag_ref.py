import sys; sys.path.insert(0,'oracle')
import pyoracle as po
ref=po.RefLib()
print('loaded', flush=True)
s=ref.build_strip(4,1,1,512); print('strip ok', flush=True)
r=ref.ldlt_serial(s,0,512); print('ldlt ok', r.det==144<<512, flush=True)
s=ref.build_strip(64,1,1,1024); print('strip64 ok', flush=True)
orc=po.OracleLib(); print(orc.ldlt(s,0,1024).det==ref.ldlt_serial(s,0,1024).det, flush=True)
