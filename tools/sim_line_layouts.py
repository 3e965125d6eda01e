"""Would a compact voxel layout cut k_fuse's DRAM reads?

A DRAM read moves whole 128-B lines (profiles/r1e_dram_granularity.txt); a
plane's line holds 16 voxels.  This host-side simulation takes one bench
keyframe (corridor, 5 mm, rendered by the reference's synth), marks the voxels
of its footprint blocks that fuse_block updates (projection inside the image,
w > 0, |dd| <= mu), and counts the 128-B lines (per plane) that hold at least
one of them under several in-block line shapes (x * y * z voxels per line).
ratio = lines * 16 / in-band voxels = read amplification of the planes.
Usage: python tools/sim_line_layouts.py [KEYFRAME_INDEX]  (needs oracle/_ref)
"""
import sys, os, numpy as np, time
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for _p in (REPO, os.path.join(REPO, 'oracle'), os.path.join(REPO, 'oracle', '_ref')):
    sys.path.insert(0, _p)
os.environ['REFUSION_BACKEND']='compiled'
import oracle as O
import refusion.synth as RS, refusion.geometry as RG
import bench as B
from paper_1709_03763_b200 import synth as SY
gt, gt_kf, dr = B.kf_poses(400)  # bench keyframe poses (ground truth)
prims=[]
for p in SY.corridor_scene():
    if p.kind==SY.ROOM: prims.append(RS.RoomShell(p.center,p.size,p.albedo))
    elif p.kind==SY.BOX: prims.append(RS.BoxSolid(p.center,p.size,p.albedo))
    else: prims.append(RS.Sphere(p.center,p.size[0],p.albedo))
scene=RS.AnalyticScene(prims); intr=RS.DEFAULT_INTRINSICS
k=int(sys.argv[1]) if len(sys.argv)>1 else 100
P=RG.Pose(gt_kf[k].rotation, gt_kf[k].translation)
t=time.time(); depth=RS.add_noise(RS.render_depth(scene,P,intr,z_max=5.0),seed=(1,7,k),sigma0=0.0015); print('render',time.time()-t)
weight=np.where(depth>0, 5/np.maximum(depth*depth,1e-12),0.0)
vs=0.005; mu=0.06
keys=O.footprint_keys(depth,weight,intr,P.rotation,P.translation,vs,mu)
coords=O.keys_to_coords(np.asarray(keys))
print('blocks',len(coords))
R=P.rotation.T; tc=P.translation
l=np.arange(512); lx=l&7; ly=(l>>3)&7; lz=l>>6
span=8*vs
res={}
inb_all=[]
for ch in range(0,len(coords),2000):
    c=np.asarray(coords[ch:ch+2000],dtype=np.float64)
    o=c*span
    vx=o[:,0:1]+(lx+0.5)*vs; vy=o[:,1:2]+(ly+0.5)*vs; vz=o[:,2:3]+(lz+0.5)*vs
    dx=vx-tc[0]; dy=vy-tc[1]; dz=vz-tc[2]
    px=R[0,0]*dx+R[0,1]*dy+R[0,2]*dz; py=R[1,0]*dx+R[1,1]*dy+R[1,2]*dz; pz=R[2,0]*dx+R[2,1]*dy+R[2,2]*dz
    with np.errstate(all='ignore'):
        u=np.floor(intr.fx*px/pz+intr.cx+0.5); v=np.floor(intr.fy*py/pz+intr.cy+0.5)
    ok=(pz>0)&(u>=0)&(u<intr.width)&(v>=0)&(v<intr.height)
    ui=np.where(ok,u,0).astype(int); vi=np.where(ok,v,0).astype(int)
    wk=weight[vi,ui]; zk=depth[vi,ui]; dd=zk-pz
    inb=ok&(wk>0)&(dd<=mu)&(dd>=-mu)
    inb_all.append(inb)
inb=np.concatenate(inb_all)  # [nblk,512]
print('voxels in band', inb.sum(), 'frac', inb.mean())
x=lx; y=ly; z=lz
layouts={
 '8x2x1 (current)': (y>>1) + 4*z,          # line id within block: 2 rows per line
 '4x4x1': (x>>2) + 2*(y>>2) + 4*z,
 '4x2x2': (x>>2) + 2*(y>>1) + 8*(z>>1),
 '2x2x4': (x>>1) + 4*(y>>1) + 16*(z>>2),
 '2x4x2': (x>>1) + 4*(y>>2) + 8*(z>>1),
}
sid=(x>>2)+2*y+16*z   # 32-B sectors: 4 x-adjacent voxels (all shapes with x-runs of 4)
S=np.zeros((512,sid.max()+1),bool); S[l,sid]=True
secs=(inb.astype(np.int32)@S.astype(np.int32))>0
print(f'sectors (4-voxel x-runs): ratio {secs.sum()*4/inb.sum():.3f}')
for name,lid in layouts.items():
    nl=lid.max()+1
    M=np.zeros((512,nl),bool); M[l,lid]=True
    lines=(inb.astype(np.int32)@M.astype(np.int32))>0
    print(f'{name:16s} lines {lines.sum():9d}  MB per plane {lines.sum()*128/1e6:7.1f}  ratio {lines.sum()*16/inb.sum():.3f}')
