"""Computable DAG (CDAG) of the n-photon Compton matrix element, and node reduction.

Build-time only (no runtime role).  Follows the paper's definitions:

* CDAG: bipartite DAG of compute nodes (pure kernel, one result) and data
  nodes (identity / transport), single exit node (§2 lines 84-88,
  App. B).
* QED kernels U (base_state), V (vertex), S1 (propagator), S2 (join), Sum
  (§2.2, App. D).
* One diagram per ordering of the N = n+1 photons on the electron line
  ((n+1)! of them, §3.1).  Each diagram is cut at the
  "tie" position j: photons 1..j are attached from the incoming electron
  (V, S1, V, ... ), photons j+1..N from the outgoing electron, and one S2
  joins the halves ("propagating one side only and multiplying the two
  sides").  Per diagram: N V, N-2 S1, 1 S2 -- which
  reproduces every Table 1 node count (SURVEY.md
  App. A.1).
* Node reduction: nodes with the same kernel and the same (ordered) parents
  are merged; children become the union (App. C, Fig. 7).
  Its fixpoint does not depend on the order; here it is
  reached by hash-consing, and ``reduce_random_order`` performs one
  reduction at a time in random order for the order-independence test.
"""
from __future__ import annotations

import itertools
import math
import random
from dataclasses import dataclass, field


@dataclass
class Node:
    kind: str                 # "data" or a compute kernel: U, V, S1, S2, Sum
    parents: list[int]        # ordered parent node ids
    label: tuple = ()         # identity of entry nodes (which external particle)
    children: set[int] = field(default_factory=set)


class CDAG:
    def __init__(self):
        self.nodes: dict[int, Node] = {}
        self._next = 0

    def add(self, kind: str, parents=(), label=()) -> int:
        nid = self._next
        self._next += 1
        self.nodes[nid] = Node(kind, list(parents), tuple(label))
        for p in parents:
            self.nodes[p].children.add(nid)
        return nid

    def compute(self, kind: str, parents, label=()) -> int:
        """Add a compute node and its single output data node; returns the data node."""
        c = self.add(kind, parents, label)
        return self.add("data", [c])

    # ------------------------------------------------------------------ stats
    def __len__(self):
        return len(self.nodes)

    def count(self, kind: str) -> int:
        return sum(1 for n in self.nodes.values() if n.kind == kind)

    def counts(self) -> dict[str, int]:
        out: dict[str, int] = {}
        for n in self.nodes.values():
            out[n.kind] = out.get(n.kind, 0) + 1
        return out

    def validate(self) -> None:
        """Bipartite, acyclic, single exit."""
        for nid, n in self.nodes.items():
            for p in n.parents:
                pk = self.nodes[p].kind
                assert (pk == "data") != (n.kind == "data"), "edge must connect data and compute"
            if n.kind == "data":
                assert len(set(n.parents)) <= 1, "data node has at most one parent"
            else:
                assert len(n.parents) >= 1
        exits = [i for i, n in self.nodes.items() if not n.children]
        assert len(exits) == 1, f"expected a single exit node, got {len(exits)}"
        # acyclic: Kahn
        indeg = {i: len(set(n.parents)) for i, n in self.nodes.items()}
        ready = [i for i, d in indeg.items() if d == 0]
        seen = 0
        while ready:
            i = ready.pop()
            seen += 1
            for c in self.nodes[i].children:
                indeg[c] -= 1
                if indeg[c] == 0:
                    ready.append(c)
        assert seen == len(self.nodes), "cycle"

    # ------------------------------------------------------------------ reduction
    def _key(self, nid: int):
        n = self.nodes[nid]
        if n.kind == "data" and not n.parents:
            return ("entry", n.label)
        return (n.kind, tuple(n.parents))

    def _merge(self, keep: int, drop: int) -> None:
        """Node reduction of two nodes with equal kernel and parents."""
        d = self.nodes.pop(drop)
        k = self.nodes[keep]
        for p in set(d.parents):
            self.nodes[p].children.discard(drop)
        for c in d.children:
            cn = self.nodes[c]
            cn.parents = [keep if p == drop else p for p in cn.parents]
            k.children.add(c)

    def reducible_groups(self) -> list[list[int]]:
        groups: dict = {}
        for nid in self.nodes:
            groups.setdefault(self._key(nid), []).append(nid)
        return [g for g in groups.values() if len(g) > 1]

    def reduce_fixpoint(self) -> "CDAG":
        """Apply node reductions until none is possible (topological sweep = hash-consing)."""
        while True:
            groups = self.reducible_groups()
            if not groups:
                return self
            for g in groups:
                g = [x for x in g if x in self.nodes]
                for d in g[1:]:
                    self._merge(g[0], d)

    def reduce_random_order(self, seed: int) -> "CDAG":
        """One reduction (merge of one maximal group) at a time, groups chosen at random."""
        rng = random.Random(seed)
        while True:
            groups = self.reducible_groups()
            if not groups:
                return self
            g = rng.choice(groups)
            for d in g[1:]:
                self._merge(g[0], d)

    def canonical(self):
        """Order-independent canonical form: each node described by its kernel and the
        canonical descriptions of its ordered parents (structural hashing)."""
        memo: dict[int, tuple] = {}

        def desc(nid):
            if nid not in memo:
                n = self.nodes[nid]
                memo[nid] = (n.kind, n.label, tuple(desc(p) for p in n.parents))
            return memo[nid]

        return sorted(hash(desc(i)) for i in self.nodes)


# ---------------------------------------------------------------------- process


@dataclass(frozen=True)
class Process:
    """e- + n_in photons -> e- + n_out photons; N = n_in + n_out photons on the line."""
    n_in_ph: int
    n_out_ph: int

    @property
    def N(self) -> int:
        return self.n_in_ph + self.n_out_ph

    @property
    def n(self) -> int:
        """The paper's / north star's n: number of photons minus one."""
        return self.N - 1

    @property
    def n_ext(self) -> int:
        return self.N + 2


def north_star(n: int) -> Process:
    """e- gamma -> e- + n gamma (BASELINE.json north_star)."""
    return Process(1, n)


def paper_process(n: int) -> Process:
    """e- gamma^n -> e- gamma."""
    return Process(n, 1)


def balanced_split(N: int) -> int:
    """Tie position j = floor(N/2) (SURVEY.md §8(c) 'tie position'; minimises the trie)."""
    return N // 2


def diagrams(N: int):
    """All N! orderings of the photons along the electron line."""
    return list(itertools.permutations(range(N)))


def build_unreduced(proc: Process, j: int | None = None) -> CDAG:
    """The generated (pre-optimisation) CDAG for fixed spins/polarisations.

    Entry data node + U per external particle; per diagram pi cut at j:
    in-side  V(eps_pi1, u) -> S1 -> V(eps_pi2, .) -> ... (j V, j-1 S1),
    out-side V(eps_piN, ubar) -> S1 -> ... (N-j V, N-j-1 S1), S2(in, out),
    and one Sum over all S2 results (App. D)."""
    N = proc.N
    if j is None:
        j = balanced_split(N)
    assert 1 <= j <= N - 1 or N == 1
    g = CDAG()
    u_in = g.compute("U", [g.add("data", label=("e_in",))])
    u_out = g.compute("U", [g.add("data", label=("e_out",))])
    eps = [g.compute("U", [g.add("data", label=("photon", i))]) for i in range(N)]
    joins = []
    for pi in diagrams(N):
        if N == 1:
            joins.append(g.compute("S2", [g.compute("V", [eps[pi[0]], u_in]), u_out]))
            continue
        left = u_in
        for l in range(j):
            if l > 0:
                left = g.compute("S1", [left])
            left = g.compute("V", [eps[pi[l]], left])
        right = u_out
        for l in range(N - j):
            if l > 0:
                right = g.compute("S1", [right])
            right = g.compute("V", [eps[pi[N - 1 - l]], right])
        joins.append(g.compute("S2", [left, right]))
    g.compute("Sum", joins)
    return g


def table1_closed_form(n: int) -> int:
    """nodes(n) = 3(n+3) + 2 + 2(2n+1)(n+1)!  (reproduces PAPER.md Table 1)."""
    return 3 * (n + 3) + 2 + 2 * (2 * n + 1) * math.factorial(n + 1)


def perm_count(N: int, i: int) -> int:
    return math.factorial(N) // math.factorial(N - i)


def reduced_counts_formula(N: int, j: int) -> dict[str, int]:
    """Counts of the fixpoint (two-sided prefix trie): V = sum_{i<=j} P(N,i) + sum_{i<=N-j} P(N,i),
    S1 = sum_{i<j} P(N,i) + sum_{i<N-j} P(N,i), S2 = N!."""
    V = sum(perm_count(N, i) for i in range(1, j + 1)) + sum(perm_count(N, i) for i in range(1, N - j + 1))
    S1 = sum(perm_count(N, i) for i in range(1, j)) + sum(perm_count(N, i) for i in range(1, N - j))
    return {"V": V, "S1": S1, "S2": math.factorial(N), "U": N + 2, "Sum": 1}
