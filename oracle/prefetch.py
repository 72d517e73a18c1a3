"""oracle.prefetch — TEST INFRASTRUCTURE ONLY. The two-resource schedule of layer-pipelined expert loading
(§4.1: "while computing the i-th layer's forward path in the compute stream, we load the
i+1-st layer's experts in a separate loading stream"), written out as SPEC.md:413-420 states it:
  * the load stream processes layers in order, one at a time (a cached layer loads in 0);
  * Prefetch: layer i's compute starts at max(compute_finish(i-1), load_finish(i));
  * OnDemand: layer i's load starts after compute_finish(i-1), its compute right after its load.
Pinned by SPEC.md's hand Gantt charts (makespans 7 / 9 / 6) in tests/test_cache.py."""


def simulate_prefetch(compute, load, mode):
    """compute[i], load[i] >= 0 per layer (load 0 = cached). Returns (starts, finishes, makespan)."""
    if len(compute) != len(load) or not compute:
        raise ValueError("need one compute and one load duration per layer, at least one layer")
    if any(c < 0 for c in compute) or any(x < 0 for x in load):
        raise ValueError("negative duration")
    starts, finishes = [], []
    load_free = 0.0      # when the load stream is next idle
    comp_free = 0.0      # compute_finish(i-1)
    for c, x in zip(compute, load):
        if mode == "prefetch":
            load_done = load_free + x
            load_free = load_done
            s = max(comp_free, load_done)
        elif mode == "on_demand":
            s = comp_free + x
        else:
            raise ValueError(mode)
        starts.append(s)
        comp_free = s + c
        finishes.append(comp_free)
    return starts, finishes, finishes[-1]
