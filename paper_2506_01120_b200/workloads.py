"""Seeded synthetic inputs for the five BASELINE configs.

Every input is generated once on the host from a fixed recipe and fed, byte
for byte, to the CUDA path, the oracle and the reference build; `digest()`
hashes what was generated so tests and bench lines can name it.

Recipes:
  * RNG: SplitMix64 with the reference's documented recurrence
    (R:include/liecl/rng.hpp:20-39), seed 0 unless stated.
  * random non-identity n-qubit string: k = next() % (4^n - 1) + 1; base-4
    digit j of k is the code (x_j | z_j << 1) of qubit j (0=I, 1=X, 2=Z,
    3=Y; the letter table of R:src/pauli.cpp:40).
  * Gaussian: Box-Muller on uniform() with 1-u inside the log.
  * dense operators come from `from_pauli` (R:src/dense.cpp:70-98): qubit 0
    is the most significant index bit, Hermitian phase i^{#Y}; a Pauli sum is
    first normalised like PauliSum::from_terms (R:src/pauli.cpp:78-115: merge
    in input order, drop |c| <= 1e-14 max|c|, sort by (z, x)).
  * generators are i*H: the i is folded into the term coefficients.

Layout: a dense operator is a d x d complex128 matrix M; its vector is the
column-major flattening vec(M)[i + j*d] = M[i, j] (Eigen storage,
R:src/dense.cpp:114-115). Tuples of operators are (count, d*d) complex128
arrays of such vectors.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

MASK64 = (1 << 64) - 1


class SplitMix64:
    """R:include/liecl/rng.hpp:20-39."""

    def __init__(self, seed: int = 0):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return float(self.next() >> 11) * (2.0 ** -53)

    def gaussian(self) -> float:
        u1, u2 = self.uniform(), self.uniform()
        return math.sqrt(-2.0 * math.log(1.0 - u1)) * math.cos(2.0 * math.pi * u2)


def random_string(rng: SplitMix64, n: int) -> tuple[int, int]:
    """Uniform non-identity n-qubit Pauli string as (x, z) masks."""
    k = rng.next() % (4 ** n - 1) + 1
    x = z = 0
    for j in range(n):
        code = (k >> (2 * j)) & 3
        x |= (code & 1) << j
        z |= (code >> 1) << j
    return x, z


@dataclass
class PauliSumSpec:
    """Normalised Pauli sum: terms sorted by (z, x), merged, dust dropped."""
    qubits: int
    x: list = field(default_factory=list)
    z: list = field(default_factory=list)
    coef: list = field(default_factory=list)  # python complex

    @staticmethod
    def from_terms(qubits: int, terms) -> "PauliSumSpec":
        acc: dict = {}
        order = []
        for (x, z), c in terms:
            key = (z, x)
            if key not in acc:
                acc[key] = complex(0.0, 0.0)
                order.append(key)
            a = acc[key]
            acc[key] = complex(a.real + c.real, a.imag + c.imag)
        max_mag = max((abs(c) for c in acc.values()), default=0.0)
        floor = 1e-14 * max_mag
        keys = sorted(k for k in acc if abs(acc[k]) > floor)
        return PauliSumSpec(qubits, [k[1] for k in keys], [k[0] for k in keys], [acc[k] for k in keys])


def _reverse_low_bits(v: int, n: int) -> int:
    r = 0
    for j in range(n):
        r |= ((v >> j) & 1) << (n - 1 - j)
    return r


def from_pauli(s: PauliSumSpec) -> np.ndarray:
    """Dense d x d expansion, R:src/dense.cpp:70-98 (same accumulation order)."""
    n = s.qubits
    d = 1 << n
    re = np.zeros((d, d))
    im = np.zeros((d, d))
    states = np.arange(d, dtype=np.uint64)
    for x, z, c in zip(s.x, s.z, s.coef):
        xi = np.uint64(_reverse_low_bits(x, n))
        zi = np.uint64(_reverse_low_bits(z, n))
        cr, ci = c.real, c.imag
        y = bin(x & z).count("1") & 3
        if y == 1:
            cr, ci = -ci, cr
        elif y == 2:
            cr, ci = -cr, -ci
        elif y == 3:
            cr, ci = ci, -cr
        parity = np.array([bin(int(v)).count("1") & 1 for v in (states & zi)], dtype=bool)
        rows = (states ^ xi).astype(np.int64)
        cols = states.astype(np.int64)
        re[rows, cols] += np.where(parity, -cr, cr)
        im[rows, cols] += np.where(parity, -ci, ci)
    return re + 1j * im


def vec(m: np.ndarray) -> np.ndarray:
    """Column-major flattening (Eigen storage order)."""
    return np.ascontiguousarray(m).ravel(order="F").astype(np.complex128)


def unvec(v: np.ndarray, d: int) -> np.ndarray:
    return np.asarray(v).reshape(d, d, order="F")


@dataclass
class DenseConfig:
    name: str
    qubits: int
    generators: np.ndarray  # (ngens, d*d) complex128, vec layout
    tol: float = 1e-10
    sums: list = field(default_factory=list)

    @property
    def d(self) -> int:
        return 1 << self.qubits

    def digest(self) -> str:
        return hashlib.sha256(np.ascontiguousarray(self.generators).tobytes()).hexdigest()


@dataclass
class PauliConfig:
    name: str
    qubits: int
    x: np.ndarray  # uint64 (ngens,)
    z: np.ndarray
    coef: np.ndarray  # (ngens, 2) float64 re/im
    tol: float = 1e-10

    def digest(self) -> str:
        h = hashlib.sha256()
        for a in (self.x, self.z, self.coef):
            h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()


I = complex(0.0, 1.0)


def _dense(name, n, sums, tol=1e-10) -> DenseConfig:
    gens = np.stack([vec(from_pauli(s)) for s in sums])
    return DenseConfig(name, n, gens, tol, sums)


# ---- the reference's HVA generator catalog (multi-term sums, §8 f2) --------

def tfim_hva_open(n: int) -> list:
    """R:src/generators.cpp:98-110: H1 = sum_i Z_i Z_{i+1} (open chain), H2 = sum_i X_i."""
    h1 = PauliSumSpec.from_terms(n, [((0, (1 << i) | (1 << (i + 1))), complex(1.0, 0.0)) for i in range(n - 1)])
    h2 = PauliSumSpec.from_terms(n, [((1 << i, 0), complex(1.0, 0.0)) for i in range(n)])
    return [h1, h2]


def xxz_hva(n: int, delta: float = 1.5) -> list:
    """R:src/generators.cpp:81-96: even- and odd-bond XX + YY + delta ZZ on the
    periodic chain (n even)."""
    def bond_sum(parity):
        terms = []
        for i in range(parity, n, 2):
            b = (1 << i) | (1 << ((i + 1) % n))
            terms += [((b, 0), complex(1.0, 0.0)), ((b, b), complex(1.0, 0.0)), ((0, b), complex(delta, 0.0))]
        return PauliSumSpec.from_terms(n, terms)
    return [bond_sum(0), bond_sum(1)]


def hea(n: int) -> list:
    """R:src/generators.cpp:37-53: X_i, Z_i, then Z_i Z_{i+1}, one term each."""
    return ([PauliSumSpec.from_terms(n, [((1 << i, 0), complex(1.0, 0.0))]) for i in range(n)] +
            [PauliSumSpec.from_terms(n, [((0, 1 << i), complex(1.0, 0.0))]) for i in range(n)] +
            [PauliSumSpec.from_terms(n, [((0, (1 << i) | (1 << (i + 1))), complex(1.0, 0.0))])
             for i in range(n - 1)])


def spin_glass_hva(n: int, seed: int = 0) -> list:
    """R:src/generators.cpp:55-77: H1 = sum_i a_i Z_i + sum_{i<j} J_ij Z_i Z_j
    (seeded uniform(-1, 1), a first, then J in (i, j) order), H2 = sum_i X_i."""
    rng = SplitMix64(seed)
    sym = lambda: 2.0 * rng.uniform() - 1.0  # uniform_symmetric, R:include/liecl/rng.hpp:36
    h1 = [((0, 1 << i), complex(sym(), 0.0)) for i in range(n)]
    h1 += [((0, (1 << i) | (1 << j)), complex(sym(), 0.0)) for i in range(n) for j in range(i + 1, n)]
    h2 = [((1 << i, 0), complex(1.0, 0.0)) for i in range(n)]
    return [PauliSumSpec.from_terms(n, h1), PauliSumSpec.from_terms(n, h2)]


def sum_arrays(sums) -> tuple:
    """(offsets, x, z, coef (t, 2)) of a list of PauliSumSpec, the C-ABI layout."""
    off, xs, zs, cs = [0], [], [], []
    for s in sums:
        xs += list(s.x)
        zs += list(s.z)
        cs += [(complex(c).real, complex(c).imag) for c in s.coef]
        off.append(len(xs))
    return (np.array(off, np.int64), np.array(xs, np.uint64), np.array(zs, np.uint64),
            np.array(cs, np.float64).reshape(-1, 2))


def config0() -> DenseConfig:
    """n=3 TFIM: i*(X0+X1+X2), i*(Z0Z1+Z1Z2) (BASELINE configs[0])."""
    n = 3
    g0 = PauliSumSpec.from_terms(n, [((1 << j, 0), I) for j in range(n)])
    g1 = PauliSumSpec.from_terms(n, [((0, (1 << j) | (1 << (j + 1))), I) for j in range(n - 1)])
    return _dense("c0_tfim_n3", n, [g0, g1])


def config1(seed: int = 0, count: int = 6) -> DenseConfig:
    """n=5: `count` generators i*P_k, P_k uniform non-identity strings."""
    n = 5
    rng = SplitMix64(seed)
    sums = [PauliSumSpec.from_terms(n, [(random_string(rng, n), I)]) for _ in range(count)]
    return _dense(f"c1_random_strings_n5_s{seed}_k{count}", n, sums)


def config2(seed: int = 0) -> DenseConfig:
    """n=6: three generators i*H_k, H_k = sum_{m<8} c_m P_m, c_m ~ N(0,1).
    Draw order per term: string, then coefficient."""
    n = 6
    rng = SplitMix64(seed)
    sums = []
    for _ in range(3):
        terms = []
        for _ in range(8):
            xz = random_string(rng, n)
            c = rng.gaussian()
            terms.append((xz, complex(0.0, c)))
        sums.append(PauliSumSpec.from_terms(n, terms))
    return _dense(f"c2_random_sums_n6_s{seed}", n, sums)


def config4() -> PauliConfig:
    """n=10 ring (bond 9-0): i*X_jX_{j+1}, i*Y_jY_{j+1}, i*Z_j, in that order."""
    n = 10
    xs, zs = [], []
    for j in range(n):
        b = (1 << j) | (1 << ((j + 1) % n))
        xs.append(b); zs.append(0)
    for j in range(n):
        b = (1 << j) | (1 << ((j + 1) % n))
        xs.append(b); zs.append(b)
    for j in range(n):
        xs.append(0); zs.append(1 << j)
    coef = np.zeros((len(xs), 2))
    coef[:, 1] = 1.0
    return PauliConfig("c4_pauli_ring_n10", n, np.array(xs, dtype=np.uint64),
                       np.array(zs, dtype=np.uint64), coef)


def pauli_config_from_strings(name: str, qubits: int, strings, coef=I) -> PauliConfig:
    xs = np.array([s[0] for s in strings], dtype=np.uint64)
    zs = np.array([s[1] for s in strings], dtype=np.uint64)
    c = np.zeros((len(strings), 2))
    c[:, 0], c[:, 1] = coef.real, coef.imag
    return PauliConfig(name, qubits, xs, zs, c)


@dataclass
class Config3:
    """Independence-check microbenchmark (BASELINE configs[3]).

    basis V = sqrt(d) * Q (Q from the QR of a seeded complex Gaussian D x N
    matrix; the sqrt(d) makes V orthonormal under <a,b> = vdot(a,b)/d,
    R:src/dense.cpp:57 -- without it every candidate would be accepted);
    candidates k even: complex Gaussian, k odd: sum_j a_j V_j + noise with
    sigma per re/im component (re, im ~ N(0,1) everywhere). 17 GB cannot
    travel, so the inputs are generated on the device with a seeded torch
    Philox generator (`generate`); the same bytes feed the CPU baseline.
    """
    d: int = 256
    n: int = 16384
    ncand: int = 4096
    noise: float = 1e-14
    seed: int = 0
    tol: float = 1e-10

    @property
    def D(self) -> int:
        return self.d * self.d

    def generate(self, torch, device):
        """-> (V (n, D) complex128, cands (ncand, D) complex128), both on `device`."""
        gen = torch.Generator(device=device)
        gen.manual_seed(self.seed)

        def cgauss(*shape):
            re = torch.randn(*shape, dtype=torch.float64, device=device, generator=gen)
            im = torch.randn(*shape, dtype=torch.float64, device=device, generator=gen)
            return torch.complex(re, im)
        G = cgauss(self.D, self.n)
        Q, _ = torch.linalg.qr(G, mode="reduced")
        del G
        V = (Q.mT * math.sqrt(self.d)).contiguous()  # row k = basis vector k (vec layout)
        del Q
        cands = torch.empty((self.ncand, self.D), dtype=torch.complex128, device=device)
        n_even = (self.ncand + 1) // 2
        cands[0::2] = cgauss(n_even, self.D)
        n_odd = self.ncand // 2
        if n_odd:
            a = cgauss(n_odd, self.n)
            cands[1::2] = a @ V + self.noise * cgauss(n_odd, self.D)
        return V, cands


@dataclass(frozen=True)
class Config3Exact:
    """Config 3's recipe at a size the reference finishes in about a minute,
    with inputs that any machine regenerates bit for bit from the seed using
    numpy alone (the reference-generated golden tests/golden/c3_exact_*.npz
    stores only the reference's outputs; the inputs are 134 MB).

    basis: V_j[e] = ph[e] * H[s_j, p(e)] / sqrt(d), with H the D x D
    Sylvester-Hadamard matrix (entries +-1), s a random row subset, p a random
    element permutation and ph a random phase in {1, i, -1, -i} per element:
    exactly orthonormal under <a, b> = vdot(a, b) / d (R:src/dense.cpp:57),
    every entry exactly (+-1 or +-i) / 8 at d = 64.
    candidates: k even complex Gaussian (PCG64 normals); k odd sum_j a_j V_j
    with dyadic a_j = round(2^10 N(0,1)) / 2^10 (every partial sum of the
    combination is an integer multiple of 2^-13 below 2^53, so any summation
    order gives the same bits), plus noise sigma = 1e-14 per re/im component
    as in config 3."""
    d: int = 64
    n: int = 2048
    ncand: int = 512
    noise: float = 1e-14
    seed: int = 7
    tol: float = 1e-10

    @property
    def D(self) -> int:
        return self.d * self.d

    @property
    def name(self) -> str:
        return f"c3_exact_d{self.d}_n{self.n}_c{self.ncand}_s{self.seed}"

    def generate_numpy(self):
        import numpy as np
        D = self.D
        rng = np.random.default_rng(self.seed)
        rows = np.sort(rng.choice(D, size=self.n, replace=False))
        perm = rng.permutation(D)
        ph = rng.integers(0, 4, size=D)
        # Sylvester-Hadamard rows: H[r, e] = (-1)^popcount(r & e)
        e = perm.astype(np.int64)
        par = np.zeros((self.n, D), np.int64)
        r = rows.astype(np.int64)[:, None]
        x = r & e[None, :]
        while np.any(x):
            par ^= x & 1
            x = x >> 1
        H = (1 - 2 * par).astype(np.float64)  # +-1, rows s_j, columns permuted
        del par, x
        re_ph = np.array([1.0, 0.0, -1.0, 0.0])[ph]
        im_ph = np.array([0.0, 1.0, 0.0, -1.0])[ph]
        scale = 1.0 / np.sqrt(self.d)  # exact for d = 4^k
        V = np.empty((self.n, D), np.complex128)
        V.real = H * (re_ph * scale)
        V.imag = H * (im_ph * scale)
        cands = np.empty((self.ncand, D), np.complex128)
        n_even = (self.ncand + 1) // 2
        g = rng.standard_normal((n_even, D, 2))
        cands[0::2].real = g[..., 0]
        cands[0::2].imag = g[..., 1]
        n_odd = self.ncand // 2
        if n_odd:
            ka = np.rint(rng.standard_normal((n_odd, self.n, 2)) * 1024.0)  # integers, |k| < 2^13
            # combination / ph = sum_j a_j H[s_j] * scale: integer sums, exact in any order
            sre = (ka[..., 0] @ H) * (scale / 1024.0)
            sim = (ka[..., 1] @ H) * (scale / 1024.0)
            # (sre + i sim) * ph with ph in {1, i, -1, -i}: exact component moves
            cre = np.where(ph == 0, sre, np.where(ph == 1, -sim, np.where(ph == 2, -sre, sim)))
            cim = np.where(ph == 0, sim, np.where(ph == 1, sre, np.where(ph == 2, -sim, -sre)))
            noise = rng.standard_normal((n_odd, D, 2)) * self.noise
            cands[1::2].real = cre + noise[..., 0]
            cands[1::2].imag = cim + noise[..., 1]
        return V, cands

    @staticmethod
    def digest(V, cands) -> str:
        import hashlib
        h = hashlib.sha256()
        h.update(V.tobytes())
        h.update(cands.tobytes())
        return h.hexdigest()[:16]
