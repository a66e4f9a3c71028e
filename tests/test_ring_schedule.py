"""CPU race / deadlock check of the ring schedule the library executes (infcl_ring_schedule: the op list of
infcl_forward and of one infcl_backward pass at world > 1; Alg.1, Alg.3, readings Q13-Q15).

n simulated ranks each enqueue their ops (several forward+backward calls back to back) on two in-order streams
(compute `st`, `comm`); a random scheduler then executes stream heads in arbitrary interleavings under the
semantics of each transport:

* IPC: a send waits (on comm) until rank r-1 has released every earlier fill of that slot, copies, then bumps
  r-1's fill counter; a wait-value blocks its stream until the slot's pairing fill has landed; a release bumps
  rank r+1's release counter (include/infcl.h);
* NCCL: a send is a grouped send(to r-1)/recv(from r+1) that completes when every rank has posted the matching
  exchange; waiting on the slot means waiting for our own exchange's event.

Every buffer carries the id of the block it holds.  Violations: a compute / send reading a buffer that does not
hold the block the schedule expects there (read before fill, stale data), a fill overwriting a slot whose current
block is still to be read (write-after-read race), or no stream able to progress (deadlock).  A mutated schedule
without the comm-stream arrival wait before forwarding (the race the multi-process GPU test once caught) must be
reported.
"""
import ctypes
import random

import pytest

from paper_2410_17243_b200 import _lib as L

OP_EVREC, OP_EVWAIT, OP_SEND, OP_WAITV, OP_RELEASE, OP_COMPUTE, OP_MERGE, OP_FINISH, OP_ALLRED = range(1, 10)
RS_ST, RS_COMM = 0, 1
XK_BLK, XK_CS, XK_LSE, XK_DT = 0, 1, 2, 3
BUF_OWN, BUF_OWNL, BUF_OWNCS, BUF_NONE = -1, -2, -3, -9


def schedule(n, r, which):
    lib = L.lib()
    cnt = lib.infcl_ring_schedule(n, r, which, None, 0)
    assert cnt > 0
    buf = (ctypes.c_int32 * (6 * cnt))()
    assert lib.infcl_ring_schedule(n, r, which, buf, cnt) == cnt
    return [tuple(buf[6 * i:6 * i + 5]) for i in range(cnt)]


class Violation(AssertionError):
    pass


def simulate(n, programs, transport, rng):
    """programs[r] = list of ops (code, a, b, c, tag).  Raises Violation on a race, stale read or deadlock."""
    # ---- host enqueue (program order): stream instances with values captured at enqueue time
    q = [[[], []] for _ in range(n)]  # q[r][stream] = list of instances
    for r in range(n):
        recs, fills, rels, sends, calls = {}, {}, {}, {}, 0
        for (code, a, b, c, tag) in programs[r]:
            if code == OP_EVREC:
                recs[b] = recs.get(b, 0) + 1
                q[r][a].append(("rec", b, recs[b]))
            elif code == OP_EVWAIT:
                q[r][a].append(("evwait", b, recs.get(b, 0)))
            elif code == OP_SEND:
                key = (a, b)
                if transport == "ipc":
                    f = fills.get(key, 0)
                    fills[key] = f + 1
                    q[r][RS_COMM].append(("send", a, b, c, tag, f, f + 1))
                else:
                    i = sends.get(key, 0)
                    sends[key] = i + 1
                    q[r][RS_COMM].append(("nsend", a, b, c, tag, i))
            elif code == OP_WAITV:
                key = (b, c)
                if transport == "ipc":
                    q[r][a].append(("waitv", b, c, fills.get(key, 0)))
                else:
                    q[r][a].append(("nwait", b, c, sends.get(key, 0)))
            elif code == OP_RELEASE:
                if transport == "ipc":
                    key = (b, c)
                    rels[key] = rels.get(key, 0) + 1
                    q[r][a].append(("release", b, c, rels[key]))
            elif code == OP_COMPUTE:
                refs = [a] + ([b] if b != BUF_NONE else [])
                q[r][RS_ST].append(("read", tuple(refs), tag))
            elif code in (OP_MERGE, OP_FINISH):
                q[r][RS_ST].append(("read", (a,), tag))
            elif code == OP_ALLRED:
                calls += 1
                q[r][RS_COMM].append(("allred", calls))
            else:
                raise AssertionError(f"unknown op {code}")
    # ---- device state
    content = [dict() for _ in range(n)]  # buffer ref -> block id; own buffers hold the rank's own block
    for r in range(n):
        for ref in (BUF_OWN, BUF_OWNL, BUF_OWNCS):
            content[r][ref] = r
    ready = [dict() for _ in range(n)]   # (kind, s) -> fill counter (IPC, written by r+1)
    freed = [dict() for _ in range(n)]   # (kind, s) -> release counter (IPC, written by r-1)
    done_ev = [dict() for _ in range(n)]
    nsent = [dict() for _ in range(n)]   # (kind, s) -> NCCL exchanges completed
    head = [[0, 0] for _ in range(n)]

    def pending_reads_expect(r, ref, blk):
        """Is a not-yet-executed instance of rank r going to read `ref` expecting block `blk`?"""
        for st in (RS_ST, RS_COMM):
            for inst in q[r][st][head[r][st]:]:
                if inst[0] == "read" and ref in inst[1] and inst[2] == blk:
                    return True
                if inst[0] in ("send", "nsend") and inst[3] == ref and inst[4] == blk:
                    return True
        return False

    def fill(r, kind, s, blk):
        ref = 2 * kind + s
        cur = content[r].get(ref)
        if cur is not None and cur != blk and pending_reads_expect(r, ref, cur):
            raise Violation(f"rank {r}: slot {(kind, s)} holding block {cur} overwritten by {blk} before it was read")
        content[r][ref] = blk

    def check_read(r, ref, blk, what):
        got = content[r].get(ref)
        if ref < 0:  # own buffers hold the rank's own block in every call
            blk = blk % n
        if got != blk:
            raise Violation(f"rank {r}: {what} reads buffer {ref} holding {got}, schedule expects block {blk}")

    def runnable(r, st):
        if head[r][st] >= len(q[r][st]):
            return False
        inst = q[r][st][head[r][st]]
        k = inst[0]
        if k == "evwait":
            return done_ev[r].get(inst[1], 0) >= inst[2]
        if k == "send":
            return freed[r].get((inst[1], inst[2]), 0) >= inst[5]
        if k == "waitv":
            return ready[r].get((inst[1], inst[2]), 0) >= inst[3]
        if k == "nwait":
            return nsent[r].get((inst[1], inst[2]), 0) >= inst[3]
        if k in ("nsend", "allred"):  # collective: every rank has the matching instance at its comm head
            for p in range(n):
                h = head[p][RS_COMM]
                if h >= len(q[p][RS_COMM]):
                    return False
                o = q[p][RS_COMM][h]
                if o[0] != k or (k == "nsend" and (o[1], o[2], o[5]) != (inst[1], inst[2], inst[5])) or \
                        (k == "allred" and o[1] != inst[1]):
                    return False
            return True
        return True

    def execute(r, st):
        inst = q[r][st][head[r][st]]
        k = inst[0]
        if k in ("nsend", "allred"):  # all ranks at once
            if k == "nsend":
                _, kind, s, _, _, _ = inst
                outs = []
                for p in range(n):
                    o = q[p][RS_COMM][head[p][RS_COMM]]
                    check_read(p, o[3], o[4], "send")
                    outs.append(o[4])
                for p in range(n):  # rank p receives what rank p+1 sent
                    fill(p, kind, s, outs[(p + 1) % n])
                    nsent[p][(kind, s)] = nsent[p].get((kind, s), 0) + 1
            for p in range(n):
                head[p][RS_COMM] += 1
            return
        head[r][st] += 1
        if k == "rec":
            done_ev[r][inst[1]] = max(done_ev[r].get(inst[1], 0), inst[2])
        elif k == "read":
            for ref in inst[1]:
                check_read(r, ref, inst[2], "compute")
        elif k == "send":
            _, kind, s, src, blk, _, v = inst
            check_read(r, src, blk, "send")
            dst = (r - 1) % n
            fill(dst, kind, s, blk)
            ready[dst][(kind, s)] = v
        elif k == "release":
            _, kind, s, v = inst
            freed[(r + 1) % n][(kind, s)] = v

    while True:
        cands = [(r, st) for r in range(n) for st in (RS_ST, RS_COMM) if runnable(r, st)]
        if not cands:
            left = sum(len(q[r][st]) - head[r][st] for r in range(n) for st in (0, 1))
            if left:
                raise Violation(f"deadlock with {left} ops pending")
            return
        execute(*rng.choice(cands))


def programs_for(n, calls, mutate=None, fused=False):
    """forward, dI pass, dT pass per call (fused: forward, one fused backward pass whose dT partials travel);
    repeated calls reuse the counters.  Block ids carried by slots are made unique per call and pass
    (id + n * phase) so a later call's read of the same slot is not mistaken for a pending read of the current
    content."""
    progs = []
    for r in range(n):
        f, b = schedule(n, r, 0), schedule(n, r, 2 if fused else 1)
        if mutate:
            f, b = mutate(f), mutate(b)
        prog = []
        for phase, ops in enumerate(([f, b] if fused else [f, b, b]) * calls):
            prog += [(c, a, bb, cc, t + n * phase if (t >= 0 and c in (OP_SEND, OP_COMPUTE, OP_MERGE, OP_FINISH))
                      else t) for (c, a, bb, cc, t) in ops]
        progs.append(prog)
    return progs


@pytest.mark.parametrize("fused", [False, True])
@pytest.mark.parametrize("transport", ["ipc", "nccl"])
@pytest.mark.parametrize("n", [2, 3, 4, 5, 8])
def test_ring_schedule_race_free(n, transport, fused):
    """Both backward schedules: the two passes, and the fused single pass whose dT partials rotate (Alg.3)."""
    rng = random.Random(1000 * n + (transport == "ipc") + 7 * fused)
    progs = programs_for(n, calls=2, fused=fused)
    for _ in range(60 if n <= 4 else 25):
        simulate(n, progs, transport, rng)


def test_fused_schedule_shape():
    """Fused backward ring: every step computes block (r + k) mod n and read-modify-writes that block's dT partial;
    the partial makes n hops (n - 1 onward + the hop home, as the forward's column state) and the call ends on the
    rank's own, complete dT."""
    for n in (2, 3, 8):
        for r in range(n):
            b = schedule(n, r, 2)
            assert [op[4] for op in b if op[0] == OP_COMPUTE] == [(r + k) % n for k in range(n)]
            assert [op[4] for op in b if op[0] == OP_MERGE] == [(r + k) % n for k in range(n)]
            assert sum(op[0] == OP_SEND and op[1] == XK_DT for op in b) == n
            assert sum(op[0] == OP_SEND and op[1] == XK_BLK for op in b) == n - 1
            assert [op for op in b if op[0] == OP_FINISH][0][4] == r


def test_checker_catches_fused_partial_race():
    """Mutation: the fused schedule without the wait for the held block's partial (read before it arrives)."""
    def drop(ops):
        return [op for op in ops if not (op[0] == OP_WAITV and op[2] == XK_DT and op[1] == RS_ST)]
    caught = 0
    for seed in range(40):
        try:
            simulate(3, programs_for(3, calls=1, mutate=drop, fused=True), "ipc", random.Random(seed))
        except Violation:
            caught += 1
    assert caught > 0


def test_schedule_shape():
    """Every step computes the block (r + k) mod n (reading Q13), the forward ends on the rank's own column
    state, and the backward pass sends n-1 blocks and n-1 LSE vectors."""
    for n in (2, 3, 8):
        for r in range(n):
            f = schedule(n, r, 0)
            assert [op[4] for op in f if op[0] == OP_COMPUTE] == [(r + k) % n for k in range(n)]
            assert [op for op in f if op[0] == OP_FINISH][0][4] == r
            assert sum(op[0] == OP_SEND and op[1] == XK_BLK for op in f) == n - 1
            assert sum(op[0] == OP_SEND and op[1] == XK_CS for op in f) == n  # + the hop home (Q15)
            b = schedule(n, r, 1)
            assert sum(op[0] == OP_SEND and op[1] == XK_LSE for op in b) == n - 1
    assert L.lib().infcl_ring_schedule(1, 0, 0, None, 0) == -1
    assert L.lib().infcl_ring_schedule(2, 0, 3, None, 0) == -1


def test_checker_catches_forwarding_before_arrival():
    """Mutation: drop the comm-stream arrival waits that guard forwarding a received block."""
    def drop(ops):
        return [op for op in ops if not (op[0] == OP_WAITV and op[1] == RS_COMM)]
    rng = random.Random(7)
    caught = 0
    for _ in range(60):
        try:
            simulate(3, programs_for(3, calls=1, mutate=drop), "ipc", rng)
        except Violation:
            caught += 1
    assert caught > 0


def test_checker_catches_missing_release():
    """Mutation: a rank that never releases its slots deadlocks its sender (IPC counters)."""
    def drop(ops):
        return [op for op in ops if op[0] != OP_RELEASE]
    with pytest.raises(Violation, match="deadlock"):
        simulate(3, programs_for(3, calls=2, mutate=drop), "ipc", random.Random(3))
