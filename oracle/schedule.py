"""Pipeline schedules of the paper, built and simulated plainly (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:93       equal number of layers per stage.
P:104-107  GPipe: all forwards, then all backwards; bubble (p-1)/m; stashes m.
P:109      PipeDream-Flush (1F1B): warm-up of differing numbers of forwards,
           steady one-forward-one-backward, drain; in-flight <= p.
P:112-118  interleaved: v model chunks per device (device 1 holds layers
           1,2,9,10 of 16 with p=4, v=2); requires m % p == 0;
           per-chunk times t_f/v, t_b/v; bubble (p-1)/(v m).

A task is a tuple (kind, mb, chunk) with kind in {"F", "B"}, 0-based
microbatch id (the figures number microbatches from 1) and chunk id.
Stage of (device r, chunk c) is sigma = c*p + r (reading of P:113).

Readings (DESIGN.md Sec. Readings): 1F1B warm-up = p - r - 1 forwards capped
at m ("differing numbers of forward passes"); interleaved order = the
group-of-p construction: forward virtual step k runs chunk (k mod pv) div p on
microbatch (k div pv)*p + k mod p; backward virtual step k runs chunk
v-1-((k mod pv) div p) on the same microbatch formula; warm-up
min(2(p-r-1) + (v-1)p, mv) forwards (with "round-robin" read as groups
of p microbatches).
"""
from fractions import Fraction
from itertools import combinations

GPIPE, ONE_F_ONE_B, INTERLEAVED = "gpipe", "1f1b", "interleaved"


class ScheduleError(ValueError):
    """Invalid (p, m, v) for a schedule kind (e.g. m % p != 0)."""


class DeadlockError(RuntimeError):
    """A static order that cannot complete under the dependency rules."""


# ----------------------------------------------------------------- stage map
def stage_map(l, p, v):
    """Layer -> (device, chunk) map.

    Stage sigma = c*p + r owns layers [sigma*Lc, (sigma+1)*Lc), Lc = l/(p v).
    Returns (dev_of_layer, chunk_of_layer) lists.  Raises ScheduleError when
    l is not divisible by p*v (equal layers per stage).
    """
    if p < 1 or v < 1 or l < 1 or l % (p * v) != 0:
        raise ScheduleError(f"l={l} not divisible by p*v={p * v}")
    Lc = l // (p * v)
    dev, chunk = [], []
    for layer in range(l):
        sigma = layer // Lc
        dev.append(sigma % p)
        chunk.append(sigma // p)
    return dev, chunk


# ---------------------------------------------------------- schedule builder
def _check(kind, p, m, v):
    if p < 1 or m < 1 or v < 1:
        raise ScheduleError("p, m, v must be >= 1")
    if kind in (GPIPE, ONE_F_ONE_B) and v != 1:
        raise ScheduleError(f"{kind} requires v == 1")
    if kind == INTERLEAVED and m % p != 0:
        raise ScheduleError(f"interleaved schedule requires m % p == 0 (P:115), got m={m}, p={p}")
    if kind not in (GPIPE, ONE_F_ONE_B, INTERLEAVED):
        raise ScheduleError(f"unknown schedule {kind!r}")


def build_schedule(kind, p, m, v, r):
    """Ordered task list of device r (2*m*v tasks)."""
    _check(kind, p, m, v)
    if not 0 <= r < p:
        raise ScheduleError(f"device {r} out of range for p={p}")
    if kind == GPIPE:
        # P:104 "forward passes for all microbatches ... followed by backward passes"
        return [("F", i, 0) for i in range(m)] + [("B", i, 0) for i in range(m)]
    if kind == ONE_F_ONE_B:
        # P:109 warm-up forwards, steady 1F1B, drain of the in-flight backwards
        warm = min(p - r - 1, m)
        order = [("F", i, 0) for i in range(warm)]
        nf, nb = warm, 0
        while nf < m:
            order.append(("F", nf, 0))
            nf += 1
            order.append(("B", nb, 0))
            nb += 1
        while nb < m:
            order.append(("B", nb, 0))
            nb += 1
        return order
    # interleaved
    total = m * v
    warm = min(2 * (p - r - 1) + (v - 1) * p, total)

    def fwd_task(k):
        g = k % (p * v)
        return ("F", (k // (p * v)) * p + k % p, g // p)

    def bwd_task(k):
        g = k % (p * v)
        return ("B", (k // (p * v)) * p + k % p, v - 1 - g // p)

    order = [fwd_task(k) for k in range(warm)]
    for i in range(total - warm):
        order.append(fwd_task(warm + i))
        order.append(bwd_task(i))
    for k in range(total - warm, total):
        order.append(bwd_task(k))
    return order


def build_all(kind, p, m, v):
    return [build_schedule(kind, p, m, v, r) for r in range(p)]


# ----------------------------------------------------------- event simulator
def _deps(task, r, p, v):
    """Cross-stage dependency of a task on device r (P:104 semantics).

    F(i, sigma) needs F(i, sigma-1); B(i, sigma) needs B(i, sigma+1), and the
    last stage's backward needs its own forward F(i, S-1).
    Returns (kind, mb, stage) or None.
    """
    kind, i, c = task
    sigma = c * p + r
    S = p * v
    if kind == "F":
        return None if sigma == 0 else ("F", i, sigma - 1)
    if sigma == S - 1:
        return ("F", i, sigma)
    return ("B", i, sigma + 1)


def simulate(orders, p, v, t_f, t_b):
    """Earliest-start execution of static per-device orders, exact rationals.

    Per-chunk durations t_f/v and t_b/v; zero communication time.
    Returns dict with 'start', 'end' {(device, task): Fraction}, 'span'.
    Raises DeadlockError when the orders cannot complete.
    """
    t_f, t_b = Fraction(t_f), Fraction(t_b)
    dur = {"F": t_f / v, "B": t_b / v}
    pos = [0] * p
    free = [Fraction(0)] * p
    done = {}  # (kind, mb, stage) -> end time
    start, end = {}, {}
    remaining = sum(len(o) for o in orders)
    while remaining:
        progressed = False
        for r in range(p):
            while pos[r] < len(orders[r]):
                task = orders[r][pos[r]]
                dep = _deps(task, r, p, v)
                if dep is not None and dep not in done:
                    break
                t0 = max(free[r], done[dep] if dep is not None else Fraction(0))
                t1 = t0 + dur[task[0]]
                kind, i, c = task
                done[(kind, i, c * p + r)] = t1
                start[(r, task)] = t0
                end[(r, task)] = t1
                free[r] = t1
                pos[r] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise DeadlockError("static orders deadlock")
    span = max(end.values()) if end else Fraction(0)
    return {"start": start, "end": end, "span": span}


def bubble_fraction(sim, m, t_f, t_b):
    """(span - m(t_f+t_b)) / (m(t_f+t_b)) (P:104-105 definition t_pb / t_id)."""
    ideal = m * (Fraction(t_f) + Fraction(t_b))
    return (sim["span"] - ideal) / ideal


def bubble_formula(kind, p, m, v):
    """(p-1)/m for GPipe and 1F1B, (p-1)/(v m) interleaved."""
    if kind == INTERLEAVED:
        return Fraction(p - 1, v * m)
    return Fraction(p - 1, m)


def peak_inflight(orders):
    """Per device: max number of (mb, chunk) whose F is done and B is not
    (P:107), counted in static order (equal to the time-based count
    since a device runs its tasks one at a time)."""
    peaks = []
    for order in orders:
        live, peak = 0, 0
        for kind, _, _ in order:
            live += 1 if kind == "F" else -1
            peak = max(peak, live)
        peaks.append(peak)
    return peaks


def validate(orders, sim, p, v, m):
    """Dependency / exclusivity checks (S:364-369 (a)-(c)); returns violations."""
    bad = []
    S = p * v
    st, en = sim["start"], sim["end"]
    where = {}
    for r, order in enumerate(orders):
        for task in order:
            kind, i, c = task
            where[(kind, i, c * p + r)] = (r, task)
    if len(where) != 2 * m * S:
        bad.append("task multiset wrong")
    for (kind, i, sigma), key in where.items():
        if kind == "F" and sigma > 0:
            if st[key] < en[where[("F", i, sigma - 1)]]:
                bad.append(("a", i, sigma))
        if kind == "B":
            dep = ("F", i, sigma) if sigma == S - 1 else ("B", i, sigma + 1)
            if st[key] < en[where[dep]]:
                bad.append(("b", i, sigma))
            if st[key] < en[where[("F", i, sigma)]]:
                bad.append(("fb", i, sigma))
    for r, order in enumerate(orders):
        for a, b in zip(order, order[1:]):
            if st[(r, b)] < en[(r, a)]:
                bad.append(("c", r))
    return bad


# ------------------------------------------------------------ channel orders
def channel_orders(orders, p, v):
    """Message order on each directed P2P channel.

    Channel ('act', r) carries activations from device r to device (r+1)%p;
    ('grad', r) carries gradients from device (r+1)%p back to device r.
    Returns {channel: (send_order, recv_order)} where each order is the list
    of (mb, sigma_of_receiving_stage) in the sequence the sender produces /
    the receiver consumes them.  FIFO channels are deadlock-free and keep the
    ideal bubble when the two orders are equal.
    """
    S = p * v
    out = {}
    if p == 1:
        return out
    for r in range(p):
        nxt = (r + 1) % p
        send_a, recv_a, send_g, recv_g = [], [], [], []
        for kind, i, c in orders[r]:
            sigma = c * p + r
            if kind == "F" and sigma < S - 1:
                send_a.append((i, sigma + 1))
        for kind, i, c in orders[nxt]:
            sigma = c * p + nxt
            if kind == "F" and sigma > 0:
                recv_a.append((i, sigma))
            if kind == "B" and sigma > 0:
                send_g.append((i, sigma - 1))
        for kind, i, c in orders[r]:
            sigma = c * p + r
            if kind == "B" and sigma < S - 1:
                recv_g.append((i, sigma))
        out[("act", r)] = (send_a, recv_a)
        out[("grad", r)] = (send_g, recv_g)
    return out


# --------------------------------------------------------------- brute force
def _merges(chains):
    """All interleavings of the given task chains (each chain keeps its order)."""
    if not chains:
        yield []
        return
    if len(chains) == 1:
        yield list(chains[0])
        return
    first, rest = chains[0], chains[1:]
    total = sum(len(c) for c in chains)
    for slots in combinations(range(total), len(first)):
        for tail in _merges(rest):
            merged, it_f, it_t = [], iter(first), iter(tail)
            sset = set(slots)
            for k in range(total):
                merged.append(next(it_f) if k in sset else next(it_t))
            yield merged


def brute_force_min_bubble(p, m, v, t_f, t_b):
    """Minimum bubble over every deadlock-free combination of per-device orders.

    Per device r the tasks of microbatch i form the chain F(i,0..v-1) then
    B(i,v-1..0) (forced by the stage dependencies); every merge of the m
    chains on every device is simulated.  Returns (min_bubble, n_combos,
    n_deadlock).  Exponential: tiny (p, m, v) only.
    """
    per_dev = []
    for r in range(p):
        chains = [[("F", i, c) for c in range(v)] + [("B", i, c) for c in reversed(range(v))]
                  for i in range(m)]
        per_dev.append(list(_merges(chains)))
    best, n, dead = None, 0, 0

    def rec(r, chosen):
        nonlocal best, n, dead
        if r == p:
            n += 1
            try:
                sim = simulate(chosen, p, v, t_f, t_b)
            except DeadlockError:
                dead += 1
                return
            bf = bubble_fraction(sim, m, t_f, t_b)
            if best is None or bf < best:
                best = bf
            return
        for o in per_dev[r]:
            rec(r + 1, chosen + [o])

    rec(0, [])
    return best, n, dead
