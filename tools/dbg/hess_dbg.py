import numpy as np
from oracle import pd_oracle as orc
from paper_2405_12484_b200 import pdsolver, material
from paper_2405_12484_b200.material import MaterialField
from paper_2405_12484_b200.volmesh import VolumeMesh
nodes = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], dtype=float)
m = VolumeMesh(nodes, np.array([[0, 1, 2, 3]])); m.node_mass = np.full(4, 0.1)
gam = MaterialField.uniform(1, 2.0, 1.0)
rng = np.random.default_rng(0)
x = nodes + 0.1 * rng.normal(size=nodes.shape)
Hd = pdsolver.exact_elastic_hessian(m, gam, x).toarray()
Ho = orc.exact_elastic_hessian(x, m.tets, m.shape_grad, m.volume, gam.gamma_s, gam.gamma_v, 4).toarray()
print("maxdiff", np.abs(Hd - Ho).max(), "scale", np.abs(Ho).max())
np.set_printoptions(precision=3, linewidth=200, suppress=True)
print(Hd[:6, :6]); print(Ho[:6, :6])
F = orc.deformation_gradients(x, m.tets, m.shape_grad)
JR, JV = material.projection_jacobians_batch(F); JRo, JVo = orc.projection_jacobians(F)
print("jac diff", np.abs(JR - JRo).max(), np.abs(JV - JVo).max())
h = pdsolver.hess_context(m, gam); h.linearize(x)
p = rng.normal(size=(4, 3))
print("apply vs oracle", np.abs(h.apply(p).reshape(-1) - Ho @ p.reshape(-1)).max())
