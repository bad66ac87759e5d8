import sys; sys.path.insert(0, "/root/repo")
import paper_2306_11148_b200 as moa
for s in [(2000,48,2000),(2048,1024,2048),(2048,2048,2048),(1920,1024,1920),(2048,512,2048),(2560,256,1920),(2600,160,2000),(7040,16,7040),(1700,1024,1408),(3000,1024,2944)]:
    pl = moa.plan(*s); print(s, pl.bm, pl.bn, pl.grid, pl.tiles, "SK" if pl.tiles > pl.grid and pl.tiles % pl.grid else "")
