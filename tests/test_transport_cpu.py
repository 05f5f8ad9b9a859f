"""Host-side logic of the multi-process hand-off on CPU (gloo, world size 2/4):
pairing, channel specs both ends must agree on, and the IPC handle exchange
protocol (the kvx IPC calls themselves need GPUs and run in the -m gpu tests)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_09334_b200.transport import ChannelSpec, exchange, pairing, role_of


def test_pairing_matches_survey_8e():
    assert pairing(2) == [(0, 1)]
    assert pairing(4) == [(0, 2), (1, 3)]
    assert pairing(8) == [(0, 4), (1, 5), (2, 6), (3, 7)]
    for bad in (0, 1, 3):
        with pytest.raises(ValueError):
            pairing(bad)


def test_roles_cover_every_rank_once():
    for world in (2, 4, 8):
        seen = {}
        for r in range(world):
            role, pair, peer = role_of(r, world)
            assert role_of(peer, world)[2] == r and role_of(peer, world)[1] == pair
            seen.setdefault(pair, set()).add(role)
        assert all(v == {"prefill", "decode"} for v in seen.values())


def test_channel_spec_layout_and_capacity():
    spec = ChannelSpec(80, 8192, 8, 128, 4, 128, 8, "pull")
    lay = spec.layout(8192)
    assert lay.fp16_bytes == 2_684_354_560  # one 4P4D pair of BASELINE config 4
    assert lay.wire_bytes == 713_031_680
    assert spec.capacity_bytes >= lay.nbytes
    assert len(spec.chunks()) == 8 and spec.chunks()[0] == (0, 10)
    assert spec.layout(100).nbytes < lay.nbytes
    with pytest.raises(ValueError):
        spec.layout(8193)
    with pytest.raises(ValueError):
        ChannelSpec(80, 8192, 8, 128, mode="rdma")
    with pytest.raises(ValueError):
        ChannelSpec(80, 8192, 8, 128, bits=3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    role, pair, peer = role_of(rank, world)
    # each rank publishes fake handles; every rank must receive its partner's
    mine = {"flags": bytes([rank]) * 64, "rank": rank, "role": role}
    if role == "prefill":
        mine["payload"] = bytes([100 + rank]) * 64
        mine["payload_off"] = 0
    allv = exchange(mine)
    theirs = allv[peer]
    ok = theirs["rank"] == peer and theirs["flags"] == bytes([peer]) * 64
    ok &= ("payload" in theirs) == (role == "decode")
    dist.barrier()
    q.put((rank, ok))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])  # 8: the 4P4D rank layout (pairs i -> i+4)
def test_handle_exchange_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res.values()) and len(res) == world


def test_pull_chunk_plan():
    from paper_2502_09334_b200.transport import pull_chunk_plan
    # config 4 pair (2.68 GB fp16): the full 8 chunks of 10 layers
    chunks, lpc = pull_chunk_plan(80, 2_684_354_560, 8, 128 << 20)
    assert lpc == 10 and len(chunks) == 8 and chunks[-1] == (70, 80)
    # a 128-token 70B-GQA prompt (42 MB): one chunk
    chunks, lpc = pull_chunk_plan(80, 41_943_040, 8, 128 << 20)
    assert chunks == [(0, 80)] and lpc == 80
    # min_chunk_bytes=0 keeps the requested chunking (tests exercise the pipeline)
    chunks, lpc = pull_chunk_plan(6, 10_000, 3, 0)
    assert chunks == [(0, 2), (2, 4), (4, 6)] and lpc == 2
    # the in-kernel doorbell rule (chunk of layer l = l // lpc) matches the list
    for L, n in ((40, 8), (33, 7), (80, 16), (5, 8)):
        chunks, lpc = pull_chunk_plan(L, 1 << 40, n, 1)
        for c, (l0, l1) in enumerate(chunks):
            assert all(l // lpc == c for l in range(l0, l1))


def test_kivi_capacity_covers_every_split():
    from hypothesis import given, settings, strategies as st

    spec = ChannelSpec(5, 300, 4, 128, 4, 32, 3, "pull", format="kivi")

    @settings(max_examples=200, deadline=None)
    @given(st.lists(st.integers(0, 300), min_size=1, max_size=16))
    def check(lens):
        total, seq = 0, []
        for n in lens:
            if total + n > 300:
                break
            seq.append(n)
            total += n
        if not seq:
            return
        assert spec.kivi_layout(seq).nbytes <= spec.capacity_bytes

    check()
    with pytest.raises(ValueError):
        ChannelSpec(5, 300, 4, 128, 4, 32, 3, "push", format="kivi")


def _geq(flag: int, value: int) -> bool:
    """The kernels' wrap-safe doorbell test (int32)(flag - value) >= 0."""
    return ((flag - value) & 0xFFFFFFFF) < (1 << 31)


def _simulate_protocol(schedule, chunks_of, Q=2, parity=False):
    """Discrete model of the pull doorbells (kvx.h sequence protocol).

    P (prefill) and D (decode) process hand-offs 1..n in order over Q queue
    slots; hand-off e publishes ``chunks_of[e - 1]`` layer chunks (the chunk
    plan depends on its token count).  Flags: ready[h][c] on D, free[h] on P;
    nothing is ever reset.  ``schedule`` picks which side tries to move next
    (one chunk per move).  Checks the safety properties at every step and
    returns (produced, consumed).  ``parity=True`` models round 1's parity
    flags (ready = p ^ 1, equality waits) for the regression test."""
    from paper_2502_09334_b200.transport import seq_of
    n = len(chunks_of)
    ready = [[0] * 64 for _ in range(Q)]
    free = [0] * Q
    published, produced, consumed = set(), [], []
    pe, pc, de, dc = 1, 0, 1, 0
    for who in schedule:
        if who == "P" and pe <= n:
            h, v = seq_of(pe, Q)
            if pc == 0:
                ok = free[h] == (v - 1) & 1 if parity else _geq(free[h], v - 1)
                if not ok:
                    continue  # P waits: D has not consumed the slot's last use
                # safe to overwrite slot h: its previous use (if any) is consumed
                assert pe <= Q or (pe - Q) in consumed
            ready[h][pc] = (v & 1) if parity else v  # parity: p ^ 1 with p = (v - 1) & 1
            published.add((pe, pc))
            pc += 1
            if pc == chunks_of[pe - 1]:
                produced.append(pe)
                pe, pc = pe + 1, 0
        elif who == "D" and de <= n:
            h, v = seq_of(de, Q)
            ok = ready[h][dc] == (v & 1) if parity else _geq(ready[h][dc], v)
            if not ok:
                continue  # K3 waits in-kernel for the doorbell
            # never reads a chunk before it is written
            assert (de, dc) in published, f"hand-off {de} chunk {dc} read before it was written"
            dc += 1
            if dc == chunks_of[de - 1]:
                consumed.append(de)
                free[h] = (v & 1) if parity else v
                de, dc = de + 1, 0
        # P never runs more than Q hand-offs ahead
        assert pe - de <= Q
    return produced, consumed


@pytest.mark.parametrize("Q", [1, 2, 3, 8])
def test_sequence_doorbells_are_safe_and_live(Q):
    """Every interleaving, hand-offs of random chunk counts (the plan follows
    the token count): no slot is overwritten before it is consumed, no chunk
    is consumed before it is produced, progress never stalls, and P can run a
    full queue (Q hand-offs) ahead of D."""
    import random
    rng = random.Random(Q)
    for trial in range(300):
        n = rng.randint(1, 4 * Q + 4)
        chunks = [rng.choice((1, 1, 2, 5, 40)) for _ in range(n)]
        sched = [rng.choice("PPD" if trial % 2 else "PDD") for _ in range(2000)]
        produced, consumed = _simulate_protocol(sched + list("PD") * 50 * n, chunks, Q)
        assert produced == list(range(1, n + 1)) and consumed == produced
    produced, _ = _simulate_protocol("P" * (Q + 3), [1] * (Q + 3), Q)
    assert produced == list(range(1, Q + 1))  # a full queue, then P waits


@pytest.mark.parametrize("Q", [1, 2])
def test_parity_doorbells_were_unsafe_for_varying_chunk_counts(Q):
    """Regression (round-1 advice): with parity flags, a long hand-off leaves
    ready[h][1..] at a parity value that the slot's use two turns later
    accepts, so D reads chunks P has not written yet.  Sequence numbers
    cannot be satisfied by an older use's flag."""
    # every slot is used long, short, long (a slot's uses are Q hand-offs apart)
    chunks = [40 if ((e - 1) // Q) % 2 == 0 else 1 for e in range(1, 3 * Q + 1)]
    sched = ("P" * 41 + "D" * 41) * (2 * len(chunks))
    with pytest.raises(AssertionError, match="read before it was written"):
        # P publishes only chunk 0 of the third use before D runs ahead
        _simulate_protocol(_lockstep(chunks), chunks, Q, parity=True)
    produced, consumed = _simulate_protocol(_lockstep(chunks), chunks, Q)
    assert consumed == list(range(1, len(chunks) + 1))
    produced, consumed = _simulate_protocol(sched, chunks, Q)
    assert consumed == list(range(1, len(chunks) + 1))


def _lockstep(chunks):
    """P publishes one chunk, then D tries to consume everything it can."""
    return ("P" + "D" * 64) * (sum(chunks) * 4)


def test_seq_of_matches_kernel_rule():
    from paper_2502_09334_b200.transport import seq_of
    # hand-off e uses slot e % Q for the v-th time
    for Q in (1, 2, 3, 8):
        uses = {}
        for e in range(1, 50):
            h, v = seq_of(e, Q)
            uses[h] = uses.get(h, 0) + 1
            assert h == e % Q and v == uses[h]
