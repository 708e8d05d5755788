"""Event-log validator — the reference's ``validate_trace`` (proj/src/trace.cpp:
94-428, contract in proj/include/totsim/trace.hpp:52-79), restated over the
device path's JSON-lines log without consulting the executor that produced it.

Checks: structure (run_begin first, run_end last, non-decreasing time); every
status change implied by node / done / reward / promote / prune records is legal
under the node lifecycle table (tree.cpp:23-45); prune counts equal the newly
tombstoned subtree; pruned nodes stay silent except late cancelled completions;
token conservation (generated == committed + reused + wasted) recomputed from
the events and matched against run_end. Problems are collected up to a cap.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

MAX_PROBLEMS = 32  # trace.cpp:71

# node lifecycle (tree.hpp:29-38) and its legal moves (tree.cpp:23-45)
PENDING, EXPANDING, AWAITING, COMMITTED, SPEC, SPEC_DONE, PRUNED, TERMINAL = range(8)
NAMES = ["PendingExpansion", "Expanding", "AwaitingReward", "Committed", "Speculative", "SpeculativeDone", "Pruned",
         "TerminalAnswer"]
LEGAL = {
    PENDING: {EXPANDING},
    EXPANDING: {AWAITING},
    AWAITING: {COMMITTED, SPEC_DONE, TERMINAL},
    SPEC: {SPEC_DONE, EXPANDING, AWAITING},  # promotion mid-flight joins the primary column
    SPEC_DONE: {COMMITTED, TERMINAL},
    COMMITTED: set(),
    TERMINAL: set(),
    PRUNED: set(),
}


def transition_legal(a: int, b: int) -> bool:
    if b == PRUNED:
        return a != PRUNED
    return b in LEGAL[a]


@dataclass
class Node:
    status: int
    spec: bool = False
    terminal: bool = False
    planned: int = 0
    done: bool = False
    rewarded: bool = False
    promoted: bool = False
    ready: int = 0
    gen: int = 0
    children: list = field(default_factory=list)


@dataclass
class Report:
    ok: bool = True
    problems: list = field(default_factory=list)
    generated: int = 0
    committed: int = 0
    reused: int = 0
    wasted: int = 0
    queries: int = 0
    makespan: float = 0.0


class _Replay:
    def __init__(self):
        self.r = Report()
        self.queries = {}  # q -> {"nodes": {id: Node}, "finished", "terminated"}
        self.requested = set()
        self.line = 0
        self.begun = False

    def flag(self, msg):
        if len(self.r.problems) < MAX_PROBLEMS:
            self.r.problems.append(f"line {self.line}: {msg}")
        self.r.ok = False

    def move(self, n: Node, to: int, why: str):
        if not transition_legal(n.status, to):
            self.flag(f"{why}: illegal transition {NAMES[n.status]} -> {NAMES[to]}")
        n.status = to

    def query(self, e):
        if "q" not in e:
            self.flag("event missing q")
            return None
        qs = self.queries.get(e["q"])
        if qs is None:
            self.flag(f"event for unadmitted query {e['q']}")
        return qs

    def node(self, qs, e):
        if "node" not in e:
            self.flag("event missing node")
            return None
        n = qs["nodes"].get(e["node"])
        if n is None:
            self.flag(f"event for undeclared node {e['node']}")
        return n

    # ---- handlers -------------------------------------------------------
    def ev_run_begin(self, e):
        if self.begun:
            self.flag("duplicate run_begin")
        self.begun = True

    def ev_admit(self, e):
        if e["q"] in self.queries:
            self.flag("query admitted twice")
            return
        self.queries[e["q"]] = {"nodes": {0: Node(COMMITTED, done=True)}, "finished": False, "terminated": False}

    def ev_node(self, e):
        qs = self.query(e)
        if qs is None:
            return
        if qs["finished"]:
            self.flag("node declared after query_done")
        nid, par = e["node"], e["parent"]
        if nid in qs["nodes"]:
            self.flag("node declared twice")
            return
        p = qs["nodes"].get(par)
        if p is None:
            self.flag("child of undeclared parent")
            return
        if p.status == PRUNED:
            self.flag("child of pruned parent")
        if e["slot"] != len(p.children):
            self.flag(f"slot {e['slot']} out of claim order")
        p.children.append(nid)
        qs["nodes"][nid] = Node(SPEC if e["spec"] else EXPANDING, spec=e["spec"], terminal=e["terminal"],
                                planned=e["tokens"])

    def ev_req(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        key = (e["q"], e["node"])
        if key in self.requested:
            self.flag("duplicate generation request for node")
        self.requested.add(key)
        if e["spec"] != n.spec:
            self.flag("request/node speculative tag mismatch")

    def ev_done(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        if n.done:
            self.flag("second completion for node")
            return
        n.done = True
        n.gen = e["tokens"]
        self.r.generated += n.gen
        if e["stale"] != (n.status == PRUNED):
            self.flag("stale flag disagrees with prune state")
        if n.status == PRUNED:
            return  # late completion of cancelled work
        if not e["cancelled"] and n.gen != n.planned:
            self.flag("full completion with unexpected token count")
        if n.spec and not n.promoted:
            if n.status != SPEC:
                self.flag(f"completion in state {NAMES[n.status]}")
        else:
            self.move(n, AWAITING, "done")

    def ev_reward(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        if n.status == PRUNED:
            self.flag("reward for pruned node")
            return
        if not n.done:
            self.flag("reward before completion")
        if n.rewarded:
            self.flag("second reward for node")
        n.rewarded = True
        if n.spec and not n.promoted:
            self.move(n, SPEC_DONE, "reward")
        else:
            self.move(n, TERMINAL if n.terminal else COMMITTED, "reward")

    def ev_promote(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        if not n.spec or n.promoted or n.status == PRUNED:
            self.flag("promote on non-promotable node")
            return
        n.promoted = True
        n.ready = e["ready"]
        if n.ready < 0 or n.ready > n.planned:
            self.flag("promote ready tokens out of range")
        if n.status == SPEC_DONE:
            if n.ready != n.gen:
                self.flag("scored promote must reuse the full generation")
            self.move(n, TERMINAL if n.terminal else COMMITTED, "promote")
        elif n.done:
            self.move(n, AWAITING, "promote")
        else:
            self.move(n, EXPANDING, "promote")

    def ev_prune(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        count, stack = 0, [e["node"]]
        while stack:
            cur = qs["nodes"][stack.pop()]
            stack.extend(cur.children)
            if cur.status == PRUNED:
                continue
            self.move(cur, PRUNED, "prune")
            count += 1
        if count != e["count"]:
            self.flag("prune count mismatch")

    def ev_answer(self, e):
        qs = self.query(e)
        n = self.node(qs, e) if qs is not None else None
        if n is None:
            return
        if not n.terminal:
            self.flag("answer from non-terminal node")
        if n.status != TERMINAL:
            self.flag("answer before terminal commit")
        if not e["weight"] >= 0.0:
            self.flag("negative answer weight")

    def ev_terminate(self, e):
        qs = self.query(e)
        if qs is None:
            return
        if qs["terminated"]:
            self.flag("query terminated twice")
        qs["terminated"] = True

    def ev_query_done(self, e):
        qs = self.query(e)
        if qs is None:
            return
        if qs["finished"]:
            self.flag("query finished twice")
            return
        qs["finished"] = True
        self.r.queries += 1
        if e["early"] and not qs["terminated"]:
            self.flag("early finish without terminate event")

    def ev_run_end(self, e):
        r = self.r
        for q in sorted(self.queries):
            qs = self.queries[q]
            if not qs["finished"]:
                self.flag(f"query {q} never finished")
            for nid in sorted(qs["nodes"]):
                if nid == 0:
                    continue
                n = qs["nodes"][nid]
                if n.status not in (COMMITTED, TERMINAL, PRUNED):
                    self.flag(f"query {q} node {nid} left in state {NAMES[n.status]}")
                useful = n.status in (COMMITTED, TERMINAL)
                if useful and not n.done:
                    self.flag("useful node without completion")
                if useful:
                    reused = n.ready if n.promoted else 0
                    r.reused += reused
                    r.committed += n.gen - reused
                else:
                    r.wasted += n.gen
        if r.generated != r.committed + r.reused + r.wasted:
            self.flag("token conservation identity broken")
        for key, mine in (("generated", r.generated), ("committed", r.committed), ("reused", r.reused),
                          ("wasted", r.wasted)):
            if e[key] != mine:
                self.flag(f"run_end {key} disagrees with replay")
        if e["queries"] != r.queries:
            self.flag("run_end queries disagrees with replay")
        r.makespan = e["makespan"]
        if abs(r.makespan - e["t"]) > 1e-9:
            self.flag("run_end timestamp disagrees with makespan")

    def run(self, events):
        if not events:
            self.flag("empty event list")
            return self.r
        if events[0].get("ev") != "run_begin":
            self.flag("first event is not run_begin")
        if events[-1].get("ev") != "run_end":
            self.flag("last event is not run_end")
        prev_t = -1.0
        for i, e in enumerate(events):
            self.line = i + 1
            if "t" not in e or "ev" not in e:
                self.flag("record missing t/ev")
                continue
            if e["t"] + 1e-12 < prev_t:
                self.flag("timestamps decrease")
            prev_t = max(prev_t, e["t"])
            h = getattr(self, "ev_" + e["ev"], None)
            if h is None:
                self.flag(f"unknown event kind: {e['ev']}")
            else:
                h(e)
            if len(self.r.problems) >= MAX_PROBLEMS:
                break
        return self.r


def validate_log(lines) -> Report:
    """validate_trace over JSON lines (str) or parsed records."""
    events = [json.loads(x) if isinstance(x, str) else x for x in lines]
    try:
        rep = _Replay().run(events)
    except (KeyError, TypeError) as ex:
        rep = Report(ok=False, problems=[f"malformed record: {ex}"])
    rep.ok = not rep.problems
    return rep
