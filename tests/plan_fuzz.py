"""Random legal pass plans (test helper): every kernel shape the C ABI
accepts -- low passes of 13/14/15 bits, one-run high passes of 1..10 rows on
the default or a forced cluster size, split-row passes -- in random order
of the lowest uncovered bit (bw_abi.cu build_passes)."""

import random


def split_entry(r, q, a, k2):
    return r | ((q + 1) << 4) | (a << 8) | (k2 << 12)


def _plain_options(r):
    """Cluster encodings legal for a one-run high pass of r rows."""
    opts = [0]  # default shape (register-only, single CTA or cluster by r)
    if 6 <= r <= 10:
        opts.append(1 << 4)  # force q = 0 (L = 13 - r in 3..7)
        opts.append(2 << 4)  # force q = 1 (L = 14 - r in 4..8)
    if 5 <= r <= 10:
        opts.append(3 << 4)  # force q = 2 (L = 15 - r in 5..10)
    return opts


def random_plan(rng: random.Random, n: int) -> list[int]:
    low = rng.choice([w for w in (13, 14, 15) if w <= n])
    plan = [low]
    covered = set(range(low))
    while len(covered) < n:
        k = min(set(range(n)) - covered)
        run = 0
        while k + run < n and (k + run) not in covered:
            run += 1
        choices = []
        for r, q in ((6, 0), (7, 0), (8, 0), (9, 1), (10, 1)):  # split-row shapes
            for a in range(1, r):
                if a > run:
                    break
                for k2 in range(k + a + 1, n - (r - a) + 1):  # a real gap between the runs
                    if all((b not in covered) for b in range(k2, k2 + r - a)):
                        choices.append(split_entry(r, q, a, k2))
        use_split = choices and rng.random() < 0.4
        if use_split:
            e = rng.choice(choices)
            r, a, k2 = e & 15, (e >> 8) & 15, (e >> 12) & 63
            covered |= set(range(k, k + a)) | set(range(k2, k2 + r - a))
            plan.append(e)
            continue
        top = min(10, run)
        r = top if rng.random() < 0.5 else rng.randint(max(1, top - 4), top)  # mostly wide passes
        plan.append(r | rng.choice(_plain_options(r)))
        covered |= set(range(k, k + r))
    return plan
