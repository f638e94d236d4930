"""CPU model check of the CASC_HALO_PEER ordering protocol (csrc/seqshard.cu apply_peer).

In the peer-halo schedule no halo is copied: the interior launch of the step producing v^(k) on
rank r stores its last rows into rank r+1's halo rows (GEMM epilogue over a peer mapping), and the
transport carries only tokens. The two ways this can go wrong are a boundary launch reading its
halo before the predecessor's push (stale rows) and a push overwriting halo rows the successor has
not finished reading (the state buffers ping-pong, so step k+1's push lands in the buffer rank r+1's
step k-1 boundary read). This test rebuilds each rank's compute-stream / comm-stream program in the
order apply_peer enqueues it, runs all ranks under randomised interleavings with NCCL's matching
rule (a grouped send/recv exchange completes once both partners reached the same exchange), and
checks: every program finishes (no deadlock), every boundary read sees the push of the same step,
and no push overwrites rows whose previous reader has not run.
"""
import random

import pytest


def programs(R, k0, kl):
    """Per rank: the compute-stream ops and comm-stream exchanges, in apply_peer's enqueue order.
    st op: (name, waits, effect); cs op: (tag, dir, waits, event). Buffers: 'a' / 'b' ping-pong."""
    buf = lambda k: "b" if k % 2 else "a"        # v^(k) lives in Va for even k (Vs of step k)  # noqa: E731
    progs = []
    for r in range(R):
        st, cs = [], []
        tag = 0
        # memsets + ev_in, then the u halo and the start token on cs
        st.append(("memset", [], ("mem", None)))
        cs.append((tag, +1, ["memset"], "uhalo")); tag += 1
        cs.append((tag, -1, ["memset"], "ack0")); tag += 1
        ack = "ack0"
        head_buf = buf(k0)
        # head: interior pushes v^(k0) into rank r+1's head buffer, boundary reads the u halo
        st.append(("int_head", [ack], ("push", head_buf, k0)))
        cs.append((tag, +1, ["int_head"], f"ready{k0}")); tag += 1
        st.append(("bnd_head", ["uhalo"], ("none", None)))
        ready = f"ready{k0}"
        for k in range(k0, kl + 1):
            if k < kl:
                st.append((f"int{k}", [ack], ("push", buf(k + 1), k + 1)))
                cs.append((tag, +1, [f"int{k}"], f"ready{k + 1}")); tag += 1
            else:
                st.append((f"int{k}", [ack], ("none", None)))
            st.append((f"bnd{k}", [ready], ("read", buf(k), k)))
            cs.append((tag, -1, [f"bnd{k}"], f"ack{k + 1}")); tag += 1
            ack = f"ack{k + 1}"
            ready = f"ready{k + 1}"
        progs.append((st, cs))
    return progs


def run(R, k0, kl, seed):
    rnd = random.Random(seed)
    progs = programs(R, k0, kl)
    pc_st, pc_cs = [0] * R, [0] * R
    done = [set() for _ in range(R)]            # completed st op names and cs events
    reached = [set() for _ in range(R)]         # exchange tags each rank has reached on cs
    halo = [dict() for _ in range(R)]           # rank -> buffer -> level last pushed into its halo
    last_read = [dict() for _ in range(R)]      # rank -> buffer -> level last read from its halo
    violations = []
    while True:
        moves = []
        for r in range(R):
            st, cs = progs[r]
            if pc_st[r] < len(st) and all(w in done[r] for w in st[pc_st[r]][1]):
                moves.append(("st", r))
            if pc_cs[r] < len(cs):
                tag, d, waits, ev = cs[pc_cs[r]]
                if all(w in done[r] for w in waits):
                    reached[r].add(tag)
                    partners = [x for x in (r + d, r - d) if 0 <= x < R]
                    if all(tag in reached[x] for x in partners):
                        moves.append(("cs", r))
        if not moves:
            break
        kind, r = rnd.choice(moves)
        if kind == "st":
            name, _, eff = progs[r][0][pc_st[r]]
            if eff[0] == "push" and r + 1 < R:
                b, lvl = eff[1], eff[2]
                prev = halo[r + 1].get(b)
                # the rows being replaced must have been read by the successor's boundary launch
                if prev is not None and last_read[r + 1].get(b) != prev:
                    violations.append(f"rank {r} pushes v^({lvl}) over unread v^({prev}) of rank {r + 1}")
                halo[r + 1][b] = lvl
            if eff[0] == "read" and r > 0:
                b, lvl = eff[1], eff[2]
                if halo[r].get(b) != lvl:
                    violations.append(f"rank {r} reads v^({lvl}) halo but holds {halo[r].get(b)}")
                last_read[r][b] = lvl
            done[r].add(name)
            pc_st[r] += 1
        else:
            done[r].add(progs[r][1][pc_cs[r]][3])
            pc_cs[r] += 1
    finished = all(pc_st[r] == len(progs[r][0]) and pc_cs[r] == len(progs[r][1]) for r in range(R))
    return finished, violations


@pytest.mark.parametrize("R", [2, 3, 4, 8])
@pytest.mark.parametrize("k0,kl", [(2, 10), (2, 2), (1, 1), (2, 5)])
def test_peer_protocol_no_deadlock_no_race(R, k0, kl):
    for seed in range(300):
        finished, violations = run(R, k0, kl, seed)
        assert finished, f"deadlock (seed {seed})"
        assert not violations, violations[:3]


def test_model_detects_a_missing_consumed_wait():
    """The check has teeth: without the consumed token before each push, some interleaving lets a
    push overwrite halo rows before the successor's boundary launch read them."""
    orig = programs

    def no_ack(R, k0, kl):
        out = []
        for st, cs in orig(R, k0, kl):
            st = [(n, [w for w in waits if not w.startswith("ack")], e) for n, waits, e in st]
            out.append((st, cs))
        return out

    globals()["programs"] = no_ack
    try:
        bad = any(run(3, 2, 8, seed)[1] for seed in range(300))
    finally:
        globals()["programs"] = orig
    assert bad
