"""Configuration space of the paper's GEMM tiling problem (oracle; test infrastructure only).

Follows PAPER.md Sec. "Problem Formulation" and "Configuration Search Modeling":

* Eq. 1-4: xi = xi_m x xi_k x xi_n, where xi_x is the set of vectors
  [x_0, ..., x_{d_x-1}] of positive integers whose product is the dimension x.
* "Multiplication of two matrices A(m x k) and B(k x n) ... m_i, k_l, n_j are the
  number of iterations of a respective loop".  Index 0 is the outermost loop (reading Z1).
* Eq. 5 + footnote: s = [s_m, s_k, s_n, J]; J true iff Eq. 2-4 hold with
  positive integers.  "Other constraints can be crafted" -> J_hw lives in ``oracle.hw``.
* Eq. 6: actions  s_x[i] <- 2 s_x[i]  and  s_x[j] <- s_x[j] / 2,
  x in {m,k,n}, i != j.
* Eq. 7: s' = step(s, a).
* Eq. 9: g(s) = [step(s,a) for all a in A]; reading Z4 keeps only the
  legitimate results, in action order (x = m,k,n; i ascending; j ascending).

A state is represented as a tuple of three tuples ``(s_m, s_k, s_n)``.
Enumeration order (reading O4, S:99-107 only asks for "a deterministic order"):
lexicographic over the concatenated factor tuple; rank = (r_m*|xi_k| + r_k)*|xi_n| + r_n.
"""
from __future__ import annotations

from math import comb
from typing import Iterator, List, Optional, Sequence, Tuple

State = Tuple[Tuple[int, ...], Tuple[int, ...], Tuple[int, ...]]
Action = Tuple[int, int, int]  # (axis index 0=m,1=k,2=n ; i doubled ; j halved)

AXES = ("m", "k", "n")


class Spec:
    """Problem instance (m, k, n, d_m, d_k, d_n) of P:172 ``cost(s; m,k,n,d_m,d_k,d_n)``.

    Note the paper's order (m, k, n); the C-ABI takes (M, N, K).
    ``family`` selects the J_hw table of ``oracle.hw`` (0 = J_prod only).
    """

    def __init__(self, m: int, k: int, n: int, dm: int = 4, dk: int = 2, dn: int = 4, family: int = 0):
        if min(m, k, n) < 1 or min(dm, dk, dn) < 1:
            raise ValueError("dimensions and depths must be >= 1 (S:30)")
        self.m, self.k, self.n = int(m), int(k), int(n)
        self.dm, self.dk, self.dn = int(dm), int(dk), int(dn)
        self.family = int(family)

    @property
    def dims(self) -> Tuple[int, int, int]:
        return (self.m, self.k, self.n)

    @property
    def depths(self) -> Tuple[int, int, int]:
        return (self.dm, self.dk, self.dn)

    def __repr__(self) -> str:
        return f"Spec(m={self.m},k={self.k},n={self.n},d=({self.dm},{self.dk},{self.dn}),family={self.family})"


# ----------------------------------------------------------------------------------------------
# Eq. 2-4: ordered factorizations of one dimension
# ----------------------------------------------------------------------------------------------

def _divisors(v: int) -> List[int]:
    return [q for q in range(1, v + 1) if v % q == 0]


def factorizations(value: int, d: int) -> List[Tuple[int, ...]]:
    """All [x_0..x_{d-1}] with positive entries and product ``value`` (Eq. 2-4), sorted
    lexicographically.  Brute force over divisors, smallest first (so the list comes out sorted)."""
    if d == 1:
        return [(value,)]
    out: List[Tuple[int, ...]] = []
    for q in _divisors(value):
        for rest in factorizations(value // q, d - 1):
            out.append((q,) + rest)
    return out


def _prime_exponents(v: int) -> List[int]:
    exps = []
    p = 2
    while p * p <= v:
        e = 0
        while v % p == 0:
            v //= p
            e += 1
        if e:
            exps.append(e)
        p += 1
    if v > 1:
        exps.append(1)
    return exps


def count_axis(value: int, d: int) -> int:
    """|xi_x| in closed form: prod over primes p^e || value of C(e + d - 1, d - 1)
    (stars and bars: the e copies of p are distributed over d ordered slots)."""
    c = 1
    for e in _prime_exponents(value):
        c *= comb(e + d - 1, d - 1)
    return c


def count_configs(spec: Spec) -> int:
    """card(xi) = |xi_m| |xi_k| |xi_n| (Eq. 1).  P:375 / P:397 print 484000, 899756, 1589952."""
    return count_axis(spec.m, spec.dm) * count_axis(spec.k, spec.dk) * count_axis(spec.n, spec.dn)


class AxisTables:
    """Per-axis sorted factorization lists plus reverse index (used by rank / unrank)."""

    def __init__(self, spec: Spec):
        self.lists = [factorizations(v, d) for v, d in zip(spec.dims, spec.depths)]
        self.index = [{t: i for i, t in enumerate(l)} for l in self.lists]
        self.card = [len(l) for l in self.lists]


_TABLE_CACHE: dict = {}


def tables(spec: Spec) -> AxisTables:
    key = (spec.dims, spec.depths)
    t = _TABLE_CACHE.get(key)
    if t is None:
        t = AxisTables(spec)
        _TABLE_CACHE[key] = t
    return t


def enumerate_configs(spec: Spec) -> Iterator[State]:
    """Every state with J_prod true exactly once, lexicographic in (m0..,k0..,n0..)."""
    t = tables(spec)
    for sm in t.lists[0]:
        for sk in t.lists[1]:
            for sn in t.lists[2]:
                yield (sm, sk, sn)


def rank(spec: Spec, s: State) -> int:
    """Position of ``s`` in ``enumerate_configs`` (mixed radix, reading O4)."""
    t = tables(spec)
    rm, rk, rn = (t.index[a][tuple(s[a])] for a in range(3))
    return (rm * t.card[1] + rk) * t.card[2] + rn


def unrank(spec: Spec, r: int) -> State:
    t = tables(spec)
    if not 0 <= r < t.card[0] * t.card[1] * t.card[2]:
        raise IndexError(r)
    rn = r % t.card[2]
    r //= t.card[2]
    rk = r % t.card[1]
    rm = r // t.card[1]
    return (t.lists[0][rm], t.lists[1][rk], t.lists[2][rn])


# ----------------------------------------------------------------------------------------------
# Eq. 5 legitimacy
# ----------------------------------------------------------------------------------------------

def j_prod(spec: Spec, s: State) -> bool:
    """P:191 footnote: Eq. 2-4 hold and all entries are positive integers."""
    if len(s) != 3:
        return False
    for a in range(3):
        vec = s[a]
        if len(vec) != spec.depths[a]:
            return False
        prod = 1
        for f in vec:
            if not isinstance(f, int) or f < 1:
                return False
            prod *= f
        if prod != spec.dims[a]:
            return False
    return True


def legitimate(spec: Spec, s: State) -> bool:
    """J = J_prod and J_hw(family) (reading Z3; "Other constraints can be crafted")."""
    if not j_prod(spec, s):
        return False
    if spec.family == 0:
        return True
    from . import hw
    return hw.j_hw(spec, s)


def initial_state(spec: Spec) -> State:
    """s0 = [[m,1,1,1],[k,1],[n,1,1,1]] "without multi-level matrix tiling"."""
    return tuple(tuple([v] + [1] * (d - 1)) for v, d in zip(spec.dims, spec.depths))  # type: ignore


# ----------------------------------------------------------------------------------------------
# Eq. 6-9: actions, step, neighbours
# ----------------------------------------------------------------------------------------------

def actions(spec: Spec) -> List[Action]:
    """A in the fixed order x = m,k,n; i ascending; j ascending, j != i.
    card = sum_x d_x (d_x - 1) = 26 at d = (4,2,4)."""
    out = []
    for a, d in enumerate(spec.depths):
        for i in range(d):
            for j in range(d):
                if i != j:
                    out.append((a, i, j))
    return out


def step(s: State, act: Action) -> Optional[State]:
    """Eq. 7 with Eq. 6's action: s_x[i] <- 2 s_x[i], s_x[j] <- s_x[j]/2.
    Returns None when s_x[j] is odd (the result would not be an integer -> J false)."""
    a, i, j = act
    vec = list(s[a])
    if vec[j] % 2 != 0:
        return None
    vec[i] *= 2
    vec[j] //= 2
    out = list(s)
    out[a] = tuple(vec)
    return tuple(out)  # type: ignore


def inverse_action(act: Action) -> Action:
    """(x, i, j) -> (x, j, i): step(step(s,a), inverse(a)) = s."""
    a, i, j = act
    return (a, j, i)


def neighbors(spec: Spec, s: State) -> List[State]:
    """g(s) (Eq. 9) restricted to legitimate results (reading Z4), in action order."""
    out = []
    for act in actions(spec):
        t = step(s, act)
        if t is not None and legitimate(spec, t):
            out.append(t)
    return out


def predecessors(spec: Spec, s2: State) -> List[Tuple[State, Action]]:
    """All (s, a) with step(s, a) = s2 and s legitimate: Alg. 2 line "for all s, for all a
    satisfying step(s,a) = s'", via s = step(s2, inverse(a))."""
    out = []
    for act in actions(spec):
        p = step(s2, inverse_action(act))
        if p is not None and legitimate(spec, p):
            out.append((p, act))
    return out


def features(spec: Spec, s: State) -> List[float]:
    """Network input: log2(f)/log2(dim) per slot; 0 when dim == 1.  The paper does
    not define an encoding (reading Z18)."""
    import math
    out = []
    for a in range(3):
        dim = spec.dims[a]
        for f in s[a]:
            out.append(0.0 if dim == 1 else math.log2(f) / math.log2(dim))
    return out


def encode(s: State) -> str:
    """Canonical text form {"m":[...],"k":[...],"n":[...]}."""
    return '{"m":[%s],"k":[%s],"n":[%s]}' % tuple(",".join(str(v) for v in s[a]) for a in range(3))


def decode(text: str, spec: Optional[Spec] = None) -> State:
    import json
    d = json.loads(text)
    if not isinstance(d, dict) or set(d) != {"m", "k", "n"}:
        raise ValueError("expected keys m, k, n")
    s = []
    for key in AXES:
        vec = d[key]
        if not isinstance(vec, list) or not all(isinstance(v, int) and not isinstance(v, bool) for v in vec):
            raise ValueError(f"non-integer entry in {key}")
        s.append(tuple(vec))
    st: State = tuple(s)  # type: ignore
    if spec is not None:
        for a in range(3):
            if len(st[a]) != spec.depths[a]:
                raise ValueError(f"axis {AXES[a]} has {len(st[a])} factors, spec wants {spec.depths[a]}")
    return st
