"""`validate` for the CUDA engine — the reference's lockstep self-check (proj/src/cli.cpp:79-140) with the
device doing the comparing.

The reference runs one scenario through two execution strategies of the same model (sequential and
thread-parallel) and requires identical state after every tick, exit code 4 on the first divergence.  The
strategies here are the engine's own: the default k-5 formulation against another one (`--variant
SFC_K5_PATH=scatter`, any SFC_* knob), the undivided grid against row slabs (`--slabs N`) or against the
band-swapped pass (`--bands N`).  Both states stay resident in HBM and are compared there every tick —
occupancy, static and dynamic images bit for bit, centres, tick (sfc_compare, the device-side
states_identical of engine.cpp:103-156) — so a 32768^2 validation never downloads an image; slab / band
variants, which run from host state, are compared on the host with states_identical.

    python -m paper_1803_04782_b200.validate scenario.scn [--ticks N] [--seed S] [--chunk-k K]
        [--variant KEY=VALUE[,KEY=VALUE...]] [--slabs N] [--bands N] [--inject-tiebreak-fault] [--every T]

Exit codes are the reference's (cli.hpp:13-18): 0 identical, 1 parse error, 2 seeding / configuration
error, 3 integrity error, 4 divergence, 5 anything else.
"""
from __future__ import annotations

import argparse
import contextlib
import os
import sys

EXIT_OK, EXIT_PARSE, EXIT_SEEDING, EXIT_INTEGRITY, EXIT_DIVERGENCE, EXIT_IO = 0, 1, 2, 3, 4, 5


@contextlib.contextmanager
def knobs(settings: dict[str, str]):
    """Engine-construction knobs (SFC_* environment variables) scoped to a block."""
    saved = {k: os.environ.get(k) for k in settings}
    os.environ.update(settings)
    try:
        yield
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def validate(sf, cfg, ticks: int, variant: dict[str, str], slabs: int = 1, bands: int = 1, fault: bool = False, every: int = 1,
             out=sys.stdout, err=sys.stderr) -> int:
    label = ", ".join([f"{k}={v}" for k, v in variant.items()] + ([f"slabs={slabs}"] if slabs > 1 else []) +
                      ([f"bands={bands}"] if bands != 1 else []) + (["tie-break fault injected"] if fault else [])) or "same configuration"
    base = sf.Engine(cfg)
    if slabs > 1 or bands != 1:  # these strategies run from host state: compare on the host, per chunk of `every` ticks
        a, b = sf.seed_population(cfg), sf.seed_population(cfg)
        with knobs(variant):
            other = sf.Engine(cfg, slabs=slabs, bands=bands, fault_invert_vote_tiebreak=fault)
        base.verify_state(a)
        done = 0
        while done < ticks:
            n = min(every, ticks - done)
            base.run(a, n)
            other.run(b, n)
            done += n
            same, why = sf.states_identical(a, b)
            if not same:
                print(f"divergence by tick {done - 1}: {why}", file=err)
                return EXIT_DIVERGENCE
    else:
        with knobs(variant):
            other = sf.Engine(cfg, fault_invert_vote_tiebreak=fault)
        base.seed_resident(cfg)
        other.seed_resident(cfg)
        done = 0
        while done < ticks:
            n = min(every, ticks - done)
            base.step_resident(n)
            other.step_resident(n)
            done += n
            same, why = base.identical_to(other)
            if not same:
                print(f"divergence at tick {done - 1} phase k-5: {why}" if every == 1 else f"divergence by tick {done - 1}: {why}", file=err)
                return EXIT_DIVERGENCE
    print(f"runs identical over {ticks} ticks ({label}); digest {base.digest() if slabs == 1 and bands == 1 else 0:#018x}", file=out)
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1803_04782_b200.validate", description=__doc__.split("\n\n")[0])
    ap.add_argument("scenario")
    ap.add_argument("--ticks", type=int)
    ap.add_argument("--seed", type=int)
    ap.add_argument("--chunk-k", type=int)
    ap.add_argument("--variant", default="", help="SFC_* knobs of the second engine, KEY=VALUE[,KEY=VALUE...]")
    ap.add_argument("--slabs", type=int, default=1)
    ap.add_argument("--bands", type=int, default=1)
    ap.add_argument("--inject-tiebreak-fault", action="store_true", help="negative control: the second engine inverts vote ties")
    ap.add_argument("--every", type=int, default=1, help="compare every this many ticks")
    args = ap.parse_args(argv)
    from paper_1803_04782_b200 import socfield as sf

    try:
        cfg = sf.parse_scenario_file(args.scenario)
        if args.ticks is not None:
            cfg.ticks = args.ticks
        if args.seed is not None:
            cfg.seed = args.seed
        if args.chunk_k is not None:
            cfg.chunk_k = args.chunk_k
        sf.validate_scenario(cfg)
        variant = dict(kv.split("=", 1) for kv in args.variant.split(",") if kv)
        return validate(sf, cfg, cfg.ticks, variant, args.slabs, args.bands, args.inject_tiebreak_fault, max(1, args.every))
    except sf.ParseError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_PARSE
    except (sf.ConfigError, sf.SeedingError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_SEEDING
    except sf.IntegrityError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INTEGRITY
    except Exception as e:  # noqa: BLE001 — the reference maps everything else to its I/O exit code
        print(f"error: {e}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
