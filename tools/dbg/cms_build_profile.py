import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2405_12484_b200 import cms, pdsolver, scenes
sc = scenes.make_scene("C3"); m = sc.mesh
K = pdsolver.assemble_global(m, sc.gammas, sc.dt).tocsr()
free = np.setdiff1d(np.arange(m.n_nodes), sc.pins)
zc = m.voxels[m.tet_voxel, 2]
labels = ((zc - zc.min()) * 8) // (zc.max() - zc.min() + 1)
Kff = K[free][:, free].tocsc()
pr = cProfile.Profile(); pr.enable()
t=time.time(); sub = cms.build_cms(Kff, m, n_domains=8, modes_per_domain=20, free=free, element_labels=labels); print('build', time.time()-t)
pr.disable(); pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
