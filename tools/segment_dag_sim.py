"""Host model of the segment-DAG sweep schedule (csrc/sk_sweep.cuh): the same
segment geometry, unit numbering, dependency counts and successor
notifications as the kernel, run as a FIFO simulation that asserts every unit
runs exactly once and only after both of its inputs (the left neighbour and
the unit of the band below that produced its alpha columns).
tests/test_host.py::test_segment_dag_model sweeps small shapes with it."""
import collections


def band_steps(rows, cols, b, H):
    return cols + min(H, rows - b * H) - 1


def seg_range(rows, cols, b, H, L):
    """(first, last) segment index of band b (SegRange in sk_sweep.cuh)."""
    return (b * H) // L, (band_steps(rows, cols, b, H) - 1 + b * H) // L


def simulate(rows, cols, npairs, slots, H=32, L=128):
    """Run the DAG; returns the number of units executed (== expected)."""
    B = (rows + H - 1) // H
    rng = [seg_range(rows, cols, b, H, L) for b in range(B)]
    spb = max(hi - lo + 1 for lo, hi in rng)
    expected = npairs * sum(hi - lo + 1 for lo, hi in rng)
    dep = collections.defaultdict(int)
    ready = collections.deque(k * B * spb for k in range(min(slots, npairs)))
    ran = set()
    while ready:
        u = ready.popleft()
        pb = u // spb
        p, b = divmod(pb, B)
        lo, hi = rng[b]
        seg = lo + (u - pb * spb)
        assert lo <= seg <= hi and (p, b, seg) not in ran
        if seg > lo:
            assert (p, b, seg - 1) in ran, ("left input", p, b, seg)
        if b > 0:  # the band below has produced every column this segment reads
            need = min(seg, rng[b - 1][1])
            assert all((p, b - 1, t) in ran for t in range(rng[b - 1][0], need + 1)), ("lower input", p, b, seg)
        ran.add((p, b, seg))
        slot_base, unit_base = (p % slots) * B * spb, p * B * spb
        if seg < hi:  # right neighbour (b, seg + 1)
            nd = 1 + (1 if b > 0 and seg + 1 <= rng[b - 1][1] else 0)
            off = b * spb + seg + 1 - lo
            dep[slot_base + off] += 1
            if dep[slot_base + off] == nd:
                ready.append(unit_base + off)
        if b + 1 < B:  # the unit above this one completes
            alo = rng[b + 1][0]
            tgt = max(seg, alo) if seg == hi else seg
            if tgt >= alo:
                nd = 1 + (1 if tgt > alo else 0)
                off = (b + 1) * spb + tgt - alo
                dep[slot_base + off] += 1
                if dep[slot_base + off] == nd:
                    ready.append(unit_base + off)
        if b + 1 == B and seg == hi and p + slots < npairs:  # slot hand-over
            for k in range(B * spb):
                dep[slot_base + k] = 0
            ready.append((p + slots) * B * spb)
    assert len(ran) == expected, ("units never ready", len(ran), expected)
    return len(ran)


if __name__ == "__main__":
    print(simulate(4095, 4095, 256, 256, L=256), simulate(300, 1, 3, 3, L=32))
