"""The paper's three benchmark environments as MDP instances (CSR, uniform |A|).

PAPER.md Sec. IV-A: FrozenLake 8x8 (64 states, 4 actions),
Taxi (500 states, 6 actions), and an N x N 2D-Maze (N = 80 / 100 gave 6166 /
9706 free cells), discount 0.95, J initialised to zero.  SURVEY 8(f) row 1.

Like the rest of gen/, this module only DEFINES instances (who goes where with
what probability and cost); it holds none of the method's arithmetic and is
shared by the CUDA path's tests and the oracle.  Readings where the paper is
silent (R22-R25):

  FrozenLake: the standard 8x8 map; slippery moves go to the intended
    direction and its two perpendiculars with 1/3 each; off-grid moves stay.
    Cost 1 per step from a normal tile; a hole costs 10^3 per step and is
    absorbing ("it will stay there with probability 1"); the goal is
    absorbing with cost 0 (a minimum-cost objective needs the goal to stop
    cost accrual).  J*(hole) = 1000 / (1 - gamma).
  Taxi: the standard 5x5 walled map, landmarks R(0,0) G(0,4) Y(4,0) B(4,3);
    state ((row*5 + col)*5 + passenger)*4 + destination (passenger 4 = in the
    taxi).  Actions 0 S, 1 N, 2 E, 3 W, 4 pick-up, 5 drop-off; deterministic.
    Cost -20 for a pick-up at the passenger's landmark and for the drop-off at
    the destination, 10 for an illegal pick-up / drop-off (a drop-off anywhere
    but the destination is illegal — with gym's "drop at another landmark"
    rule a -20 pick-up could be farmed forever), 1 otherwise (a move into a
    wall keeps the taxi in place at cost 1).  A delivered passenger
    (passenger == destination) is absorbing at cost 0.
  Maze: obstacles on ~3.5 % of the cells (hashed from the seed), every free
    cell not connected to the terminal (the bottom-right cell) becomes an
    obstacle; the free cells are the states.  Moves: slip 0.7 to the intended
    neighbour (blocked -> stay), the remaining 0.3 uniform over staying and
    the other admissible neighbours — every admissible (state, action, next
    state) triple has non-null probability.  Cost 1, terminal 0 and
    absorbing.
"""
from __future__ import annotations

from collections import deque

import numpy as np

FROZENLAKE_8x8 = [
    "SFFFFFFF",
    "FFFFFFFF",
    "FFFHFFFF",
    "FFFFFHFF",
    "FFFHFFFF",
    "FHHFFFHF",
    "FHFFHFHF",
    "FFFHFFFG",
]

TAXI_MAP = [
    "+---------+",
    "|R: | : :G|",
    "| : | : : |",
    "| : : : : |",
    "| | : | : |",
    "|Y| : |B: |",
    "+---------+",
]
TAXI_LOCS = [(0, 0), (0, 4), (4, 0), (4, 3)]


def _to_csr(rows, n, A, dtype):
    """rows[s][a] = (dict next_state -> probability, cost) -> (row_ptr, col, val, c)."""
    row_ptr = np.zeros(n * A + 1, dtype=np.int64)
    cols, vals = [], []
    c = np.zeros((n, A), dtype=dtype)
    for s in range(n):
        for a in range(A):
            succ, cost = rows[s][a]
            ks = sorted(succ)
            cols.extend(ks)
            vals.extend(succ[k] for k in ks)
            row_ptr[s * A + a + 1] = row_ptr[s * A + a] + len(ks)
            c[s, a] = cost
    return row_ptr, np.asarray(cols, dtype=np.int32), np.asarray(vals, dtype=dtype), c


def frozenlake(dtype=np.float64):
    """FrozenLake 8x8: (n=64, A=4, row_ptr, col, val, c, info)."""
    grid = FROZENLAKE_8x8
    N = len(grid)
    n, A = N * N, 4
    moves = [(0, -1), (1, 0), (0, 1), (-1, 0)]  # (dr, dq): 0 left, 1 down, 2 right, 3 up (gym order)
    rows = []
    for s in range(n):
        r, q = divmod(s, N)
        tile = grid[r][q]
        acts = []
        for a in range(A):
            if tile in "HG":
                acts.append(({s: 1.0}, 1000.0 if tile == "H" else 0.0))
                continue
            succ = {}
            for b in ((a - 1) % 4, a, (a + 1) % 4):
                dr, dq = moves[b]
                rr, qq = r + dr, q + dq
                t = rr * N + qq if 0 <= rr < N and 0 <= qq < N else s
                succ[t] = succ.get(t, 0.0) + 1.0 / 3.0
            acts.append((succ, 1.0))
        rows.append(acts)
    holes = [s for s in range(n) if grid[s // N][s % N] == "H"]
    goal = [s for s in range(n) if grid[s // N][s % N] == "G"]
    return (n, A) + _to_csr(rows, n, A, dtype) + ({"holes": holes, "goal": goal},)


def _taxi_blocked(r, q, dq):
    """True if a move east (dq=+1) / west (dq=-1) from (r, q) hits a wall."""
    line = TAXI_MAP[r + 1]
    x = 2 * q + 1 + dq  # the separator between the cells
    return line[x] == "|"


def taxi_state(r, q, p, d):
    return ((r * 5 + q) * 5 + p) * 4 + d


def taxi(dtype=np.float64):
    """Taxi: (n=500, A=6, row_ptr, col, val, c, info)."""
    n, A = 500, 6
    rows = []
    for s in range(n):
        d = s % 4
        p = (s // 4) % 5
        q = (s // 20) % 5
        r = s // 100
        acts = []
        if p == d:  # delivered: absorbing, cost 0
            rows.append([({s: 1.0}, 0.0)] * A)
            continue
        for a in range(A):
            nr, nq, np_, cost = r, q, p, 1.0
            if a == 0:
                nr = min(r + 1, 4)
            elif a == 1:
                nr = max(r - 1, 0)
            elif a == 2:
                if q < 4 and not _taxi_blocked(r, q, +1):
                    nq = q + 1
            elif a == 3:
                if q > 0 and not _taxi_blocked(r, q, -1):
                    nq = q - 1
            elif a == 4:
                if p < 4 and TAXI_LOCS[p] == (r, q):
                    np_, cost = 4, -20.0
                else:
                    cost = 10.0
            else:
                if p == 4 and TAXI_LOCS[d] == (r, q):
                    np_, cost = d, -20.0
                else:
                    cost = 10.0
            acts.append(({taxi_state(nr, nq, np_, d): 1.0}, cost))
        rows.append(acts)
    terminal = [s for s in range(n) if (s // 4) % 5 == s % 4]
    return (n, A) + _to_csr(rows, n, A, dtype) + ({"terminal": terminal},)


def _mix(z):
    z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return z ^ (z >> 31)


def maze(N, seed=1, density=0.035, slip=0.7, dtype=np.float64):
    """N x N maze: (n, A=4, row_ptr, col, val, c, info) over the free cells."""
    free = np.ones((N, N), dtype=bool)
    thr = int(density * 2**64)
    for r in range(N):
        for q in range(N):
            if _mix(_mix(seed ^ 0x4D415A45) ^ (r * N + q)) < thr:
                free[r, q] = False
    goal = (N - 1, N - 1)
    free[goal] = True
    # keep only the cells connected to the terminal
    seen = np.zeros_like(free)
    dq_ = deque([goal])
    seen[goal] = True
    while dq_:
        r, q = dq_.popleft()
        for dr, dc in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            rr, qq = r + dr, q + dc
            if 0 <= rr < N and 0 <= qq < N and free[rr, qq] and not seen[rr, qq]:
                seen[rr, qq] = True
                dq_.append((rr, qq))
    free &= seen
    cells = [(r, q) for r in range(N) for q in range(N) if free[r, q]]
    index = {cell: i for i, cell in enumerate(cells)}
    n, A = len(cells), 4
    moves = [(-1, 0), (1, 0), (0, -1), (0, 1)]  # 0 N, 1 S, 2 W, 3 E
    t = index[goal]
    rows = []
    for i, (r, q) in enumerate(cells):
        if i == t:
            rows.append([({i: 1.0}, 0.0)] * A)
            continue
        nb = []
        for dr, dc in moves:
            cell = (r + dr, q + dc)
            nb.append(index.get(cell))
        acts = []
        for a in range(A):
            others = [nb[b] for b in range(A) if b != a and nb[b] is not None]
            p_other = (1.0 - slip) / (1 + len(others))
            succ = {i: p_other}
            tgt = nb[a] if nb[a] is not None else i
            succ[tgt] = succ.get(tgt, 0.0) + slip
            for o in others:
                succ[o] = succ.get(o, 0.0) + p_other
            acts.append((succ, 1.0))
        rows.append(acts)
    return (n, A) + _to_csr(rows, n, A, dtype) + ({"terminal": t, "N": N, "free": free},)


def dense_from_csr(n, A, row_ptr, col, val):
    """Scatter a CSR instance into a dense [n][A][n] array of val's dtype."""
    P = np.zeros((n * A, n), dtype=val.dtype)
    for r in range(n * A):
        for e in range(row_ptr[r], row_ptr[r + 1]):
            P[r, col[e]] += val[e]
    return P.reshape(n, A, n)
