import sys, numpy as np, dataclasses
sys.path.insert(0,'/root/repo')
from oracle import ts_oracle as O
R,S,s=128,1024,100.0
og=O.build_grid(R); of=O.init_sphere_field(og)
active=O.prefilter(og,of,s)
cam=O.orbit_camera(1,8,width=S,height=S)
sc=O.build_scene(og,of,cam,s,active=active)
b=O.bin_and_sort(sc,cam)
m1,_=O.render_forward(sc,b,cam,want_counts=True)
rng=np.random.default_rng(0)
d2=sc.depths.copy()
mask=rng.uniform(size=d2.shape)<0.2
d2[mask]=np.nextafter(d2[mask], np.where(rng.uniform(size=mask.sum())<0.5, -np.inf, np.inf))
md2=d2.mean(axis=1)
print("md changed", (md2!=sc.mean_depth).mean())
sc2=dataclasses.replace(sc, depths=d2, mean_depth=md2)
b2=O.bin_and_sort(sc2,cam)
print("items same", np.array_equal(b2.items,b.items))
m2,_=O.render_forward(sc2,b2,cam,want_counts=True)
for k in ("normal","depth","opacity"):
    a,r=getattr(m2,k),getattr(m1,k)
    e=np.abs(a-r)
    print(k, e.max()/np.abs(r).max(), np.unravel_index(np.argmax(e if e.ndim==2 else e.max(2)), r.shape[:2]))
