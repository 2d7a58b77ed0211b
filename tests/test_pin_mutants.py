"""The pins bite: each round-2 pin (tests/test_oracle_pins_r2.py) is re-run against a
deliberately broken copy of the oracle (one source line mutated, loaded as a fresh module)
and must FAIL there.  A pin that also passes on a mutant would not catch that mistake."""
import os
import sys
import types

import pytest

import tests.test_oracle_pins_r2 as pins

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_mutant(modname, old, new):
    """oracle/<modname>.py with `old` replaced by `new` (exactly once), as a new module."""
    path = os.path.join(ROOT, "oracle", modname + ".py")
    src = open(path).read()
    assert src.count(old) == 1, f"mutation anchor not unique in oracle/{modname}.py: {old!r}"
    name = f"oracle._mutant_{modname}"
    mod = types.ModuleType(name)
    mod.__package__ = "oracle"
    mod.__file__ = path
    sys.modules[name] = mod
    exec(compile(src.replace(old, new), path, "exec"), mod.__dict__)
    return mod


def run_pin(monkeypatch, search=None, schedule=None, fn=None, *args):
    if search is not None:
        for nm in ("OracleTuner", "Space", "table_cost"):
            monkeypatch.setattr(pins, nm, getattr(search, nm))
    if schedule is not None:
        monkeypatch.setattr(pins, "oschedule", schedule.schedule)
    fn(*args)


SEARCH_MUTANTS = [
    # (description, old, new, pin, args)
    ("rejected draws re-draw only the knobs (sketch drawn once per call)",
     "            s = self.rng.uniform(self.space.nsketch)\n",
     "            s = self.rng.uniform(self.space.nsketch) if attempts == 1 else s\n",
     pins.test_sampler_hand_traced_with_rejected_draw, ()),
    ("attempt cap 32 n instead of 64 n",
     "while len(out) < n and attempts < 64 * n:", "while len(out) < n and attempts < 32 * n:",
     pins.test_sampler_duplicates_consume_output_until_the_cap, ()),
    ("knob drawn before the sketch",
     "            s = self.rng.uniform(self.space.nsketch)\n            idx = tuple(self.rng.uniform(c) for c in self.space.cards(s))\n",
     "            _u = self.rng.next()\n            s = self.rng.uniform(self.space.nsketch)\n            idx = tuple((_u * c) >> 64 for c in self.space.cards(s))\n",
     pins.test_sampler_hand_traced_with_rejected_draw, ()),
    ("alpha gate ignored", "return alpha <= 0 or wilcoxon_p(self.smemo[p], self.smemo[q]) < alpha",
     "return True", pins.test_alpha_gate_spec_worked_example, (0.05, False)),
    ("alpha gate <= instead of <", "return alpha <= 0 or wilcoxon_p(self.smemo[p], self.smemo[q]) < alpha",
     "return alpha <= 0 or wilcoxon_p(self.smemo[p], self.smemo[q]) <= alpha",
     pins.test_alpha_gate_spec_worked_example, (0.1, False)),
    ("GROW ray from the new point instead of the previous one",
     "i = min(max(prev[1][d] + step * (2 ** j), 0), card - 1)", "i = min(max(x[1][d] + step * (2 ** j), 0), card - 1)",
     pins.test_grow_closed_form_counts, ()),
    ("ties go to the last ring point", "if best_p is None or self.memo[p] < best_c:",
     "if best_p is None or self.memo[p] <= best_c:", pins.test_plain_closed_form_counts, ()),
]


@pytest.mark.parametrize("desc,old,new,pin,args", SEARCH_MUTANTS, ids=[m[0] for m in SEARCH_MUTANTS])
def test_search_pins_fail_on_mutants(monkeypatch, desc, old, new, pin, args):
    mut = load_mutant("search", old, new)
    with pytest.raises(AssertionError):
        run_pin(monkeypatch, mut, None, pin, *args)


SCHEDULE_MUTANTS = [
    ("drop rule deleted",
     "        work = [i for i in work if not (math.isfinite(wbest(i)) and wbest(i) < drop_frac * model)]\n", "",
     (0.1, 1.0, [4, 4, 30])),
    ("drop ignores the layer weight",
     "wbest(i) < drop_frac * model)]", "tuners[i].best()[1] < drop_frac * model)]", (0.1, 100.0, [4, 4, 64])),
    ("drop compares with the largest layer, not the model total",
     "        model = sum(wbest(i) for i in range(L) if math.isfinite(wbest(i)))\n",
     "        model = max(wbest(i) for i in range(L) if math.isfinite(wbest(i))) * 100\n",
     (10.0, 1.0, [4, 4, 64])),
]


@pytest.mark.parametrize("desc,old,new,args", SCHEDULE_MUTANTS, ids=[m[0] for m in SCHEDULE_MUTANTS])
def test_schedule_pins_fail_on_mutants(monkeypatch, desc, old, new, args):
    mut = load_mutant("schedule", old, new)
    with pytest.raises(AssertionError):
        run_pin(monkeypatch, None, mut, pins.test_drop_rule_hand_derived, *args)


def test_unmutated_oracle_passes_the_same_harness(monkeypatch):
    # control: the harness itself does not manufacture failures
    same = load_mutant("search", "MASK64 = (1 << 64) - 1", "MASK64 = (1 << 64) - 1")
    run_pin(monkeypatch, same, None, pins.test_sampler_hand_traced_with_rejected_draw)
    run_pin(monkeypatch, same, None, pins.test_grow_closed_form_counts)
    sch = load_mutant("schedule", "import math", "import math")
    run_pin(monkeypatch, same, sch, pins.test_drop_rule_hand_derived, 0.1, 1.0, [4, 4, 30])
