import sys, os
sys.path.insert(0, os.getcwd())
from paper_2506_01120_b200 import liecl
X, Z = liecl.PauliString(1, 0, 1), liecl.PauliString(0, 1, 1)
gens = [liecl.pauli_sum_from_terms(1, [(X, 1.0)]), liecl.pauli_sum_from_terms(1, [(Z, 1.0)])]
res = liecl.run_closure(gens, liecl.Method.orthonorm_dimonly, liecl.ClosureConfig(tolerance=1e-10))
print(res.dimension)
print(liecl.basis_listing(res))
dense = liecl.from_pauli(gens)
res2 = liecl.run_closure(dense, liecl.Method.matrix_inversion)
print(res2.dimension, res2.gram[0].shape)
