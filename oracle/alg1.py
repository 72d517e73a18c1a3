"""oracle.alg1 — TEST INFRASTRUCTURE ONLY. Alg. 1 (expert-aware batching, §4.2) written
line by line in plain Python over per-expert FIFO lists, with the two readings of DESIGN.md Q12:
`ReqQueueByExpert[k]` (lines 250, 256-257, stale loop variable) is read as `ReqQueueByExpert[E]`, and the
loop stops when the largest queue is empty (the pseudocode never terminates otherwise). argmax ties go to
the lowest expert id."""


def schedule(queues, max_token_len):
    """queues: list of lists (token ids per expert, FIFO). Returns (scheduled [(token, expert)], new queues)."""
    queues = [list(q) for q in queues]
    num_experts = len(queues)
    len_reqs_per_experts = [0] * num_experts
    for k in range(num_experts):                                   # lines 1-3
        len_reqs_per_experts[k] = len(queues[k])
    scheduled = []
    while True:                                                    # line 4
        E = max(range(num_experts), key=lambda e: (len_reqs_per_experts[e], -e))  # line 5
        if len_reqs_per_experts[E] == 0:                           # reading Q12: termination
            break
        if len_reqs_per_experts[E] < (max_token_len - len(scheduled)):   # line 6
            scheduled += [(t, E) for t in queues[E]]               # line 7
            queues[E] = []                                         # line 8
            len_reqs_per_experts[E] = 0                            # line 9
        elif max_token_len - len(scheduled) >= 0:                  # line 10
            n_available = max_token_len - len(scheduled)           # line 11
            scheduled += [(t, E) for t in queues[E][:n_available]]  # line 12
            queues[E] = queues[E][n_available:]                    # line 13
            len_reqs_per_experts[E] = len(queues[E])               # line 14
            break                                                  # line 15
        else:
            break                                                  # line 17
    return scheduled, queues
