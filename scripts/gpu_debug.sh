python - <<'PY'
import numpy as np, paper_2106_04487_b200 as fkt
from oracle import ref
for d in (2,3,4,5):
  for name in ("exponential","cauchy","gaussian","matern32"):
    x,y=fkt.synthCloud("cube",1500,d,100+d)
    k=fkt.makeKernel(name)
    p=fkt.plan(fkt.PointCloud.from_array(x),k,fkt.FktOptions(p=4,theta=0.75,leafCapacity=128))
    z=p.multiply(y); zd=fkt.denseMultiply(fkt.PointCloud.from_array(x),k,y)
    zr=ref.dense(x,name,{},y); rp=ref.RefPlan(x,name,{},p=4,theta=0.75,leaf=128); zf=rp.multiply(y)
    print(d,name,"fkt-vs-dense",fkt.relativeError(z,zd),"gpu dense vs ref dense",fkt.relativeError(zd,zr),"ref fkt vs dense",fkt.relativeError(zf,zr))
PY
