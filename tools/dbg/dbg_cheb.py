import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
from oracle import pd_oracle as orc
from paper_2405_12484_b200 import cms as gcms, scenes, _abi
from pdtest_helpers import golden
sc = scenes.c1_swatch(); m = sc.mesh
K = orc.assemble_K(m.tets, m.shape_grad, m.volume, sc.gammas.gamma_s, sc.gammas.gamma_v, m.node_mass, sc.dt, sc.n_nodes)
free = np.setdiff1d(np.arange(sc.n_nodes), sc.pins); Kff = K[free][:, free].tocsc()
g = golden("solvers.npz")
rho_o = orc.power_rho(Kff, 1.0/Kff.diagonal(), 0.75)
ctx = _abi.MatrixContext(Kff, np.empty(0, dtype=np.int64))
rho_g = gcms._power_rho(ctx, Kff.shape[0], 0.75)
print("rho oracle", rho_o, "gpu", rho_g)
x_o, info_o = orc.a_jacobi_refine(Kff, g["b"], g["x0"], sweeps=10, aggregation=2, chebyshev=True, rho=rho_o)
x_g, info_g = gcms.a_jacobi_refine(Kff, g["b"], g["x0"], sweeps=10, aggregation=2, chebyshev=True, rho=rho_o)
print("x diff", np.abs(x_o-x_g).max(), "golden diff", np.abs(x_o-g["cheb_x"]).max())
print(np.array(info_o["residuals"][:6])); print(np.array(info_g["residuals"][:6]))
