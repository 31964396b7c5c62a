"""O4 — Selective CUDA Graphs: the cost-benefit rule.

Per segment the slow path measures, in microseconds:
  L   host launch cost per kernel        d_k  device time of kernel k
  G   host cudaGraphLaunch cost          delta per-node in-graph overhead
  c_copy, c_ind   rebinding cost of the COPY / INDIRECT arms (SURVEY §8(d) Δ)
and optionally the three measured end-to-end totals ("runs each of the available modules
..., measures their execution time, and caches the module with the best performance").

Estimates (IEEE double, left-to-right, same order as the C library so decisions are bit-exact):
  eager   SPEC two-resource recurrence:
            issue_k = k*L (k = 1..K); start_k = max(free, issue_k); free = start_k + d_k
  graph   t_graph = G + sum_k (delta + d_k) [+ F]   (S:L413 minus prelude/RNG; F = fixed
          per-replay overhead, e.g. SPEC's host_obj_rebuild, default 0)
  t_copy = t_graph + c_copy;  t_ind = t_graph + c_ind
Decision: argmin over [t_eager, t_copy, t_ind] scanned in that order with strict '<', so ties go
EAGER > COPY > INDIRECT (ambiguity 8). INDIRECT drops out when unavailable.

Model 1 (p["model"] == 1): the replay the runtime actually deploys is the chain's dependency DAG
(DESIGN §5), not a serial sequence, so t_graph = G + sum(delta + d_k) no longer describes it (fitting
delta to a DAG replay gave negative values). Its replay is a list schedule of the DAG in
chain (issue) order:
            issue_k = (k + 1) * delta                   (the graph executor's issue interval)
            start_k = max(issue_k, max_{j in deps(k)} fin_j + lam)   (lam: dependency latency)
            fin_k   = start_k + g_k                     (g_k: the node's work time in that replay)
            S       = max_k fin_k
            t_graph = max(G, S) + F
        with max(G, S) because back-to-back replays overlap the host launch of replay i+1 with
        the device work of replay i (the two-resource reasoning of the eager recurrence, S:L404,
        applied to whole replays; DESIGN §3 reading 15). For a linear chain with lam == delta and
        G == 0 this is exactly the serial form sum_k (delta + g_k) + F (pinned in the tests).
"""
from __future__ import annotations

EAGER, GRAPH_COPY, GRAPH_INDIRECT = 0, 1, 2
NAMES = {EAGER: "EAGER", GRAPH_COPY: "GRAPH_COPY", GRAPH_INDIRECT: "GRAPH_INDIRECT"}


def t_eager(L: float, d) -> float:
    """SPEC S:L404 two-resource pipeline; examples S:L408-409 (110 us, 1005 us)."""
    free = 0.0
    for k, dk in enumerate(d, start=1):
        issue = k * L
        start = free if free > issue else issue
        free = start + dk
    return free


def t_graph(G: float, delta: float, d, F: float = 0.0) -> float:
    """Replay core: G + sum_k (delta + d_k) + F, summed left to right."""
    s = G
    for dk in d:
        s = s + (delta + dk)
    return s + F


def t_graph_dag(G: float, delta: float, lam: float, g, deps, F: float = 0.0) -> float:
    """Model 1: list schedule of the dependency DAG (module docstring). deps[k] lists the indices
    j < k the k-th node depends on. Same operation order as the C library (bit-exact)."""
    fin = []
    S = 0.0
    for k, gk in enumerate(g):
        start = (k + 1) * delta
        for j in deps[k]:
            c = fin[j] + lam
            if c > start:
                start = c
        f = start + gk
        fin.append(f)
        if f > S:
            S = f
    return (G if G > S else S) + F


def estimates(p: dict) -> tuple:
    """(t_eager, t_copy, t_ind) from a profile dict with keys L, G, delta, d, c_copy, c_ind [, F];
    model 1 also lam, g, deps."""
    if p.get("model", 0) == 1:
        tg = t_graph_dag(p["G"], p["delta"], p["lam"], p["g"], p["deps"], p.get("F", 0.0))
    else:
        tg = t_graph(p["G"], p["delta"], p["d"], p.get("F", 0.0))
    return t_eager(p["L"], p["d"]), tg + p["c_copy"], tg + p["c_ind"]


def decide(t_e: float, t_c: float, t_i: float, ind_available: bool = True) -> int:
    """Three-way argmin with strict '<' in the fixed order EAGER, COPY, INDIRECT."""
    best, bt = EAGER, t_e
    if t_c < bt:
        best, bt = GRAPH_COPY, t_c
    if ind_available and t_i < bt:
        best, bt = GRAPH_INDIRECT, t_i
    return best


def select(profiles: list) -> list:
    """Per-segment decisions, each independent of the others."""
    out = []
    for p in profiles:
        if p.get("use_measured", False):
            t = (p["t_eager"], p["t_copy"], p["t_ind"])
        else:
            t = estimates(p)
        out.append(decide(*t, ind_available=p.get("ind_available", True)))
    return out
