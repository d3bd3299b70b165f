"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) by kernel."""
import collections
import csv
import re
import sys


def load(path):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    seq = []
    for r in rows[1:]:
        if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[idx["Metric Value"]].replace(",", ""))
        unit = r[idx["Metric Unit"]]
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
        name = re.sub(r"\(.*", "", r[idx["Kernel Name"]])
        name = re.sub(r"^void ", "", name)
        seq.append((name[:70], v, r[idx["Grid Size"]], r[idx["Block Size"]]))
    return seq


def summarize(seq, title=""):
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for n, v, _, _ in seq:
        tot[n] += v
        cnt[n] += 1
    total = sum(tot.values())
    print(f"== {title}: {len(seq)} launches, {total / 1e3:.3f} ms")
    for n in sorted(tot, key=lambda k: -tot[k])[:20]:
        print("%-70s %5d %10.1f us %5.1f%%  avg %8.2f us" % (n, cnt[n], tot[n], 100 * tot[n] / total, tot[n] / cnt[n]))


if __name__ == "__main__":
    seq = load(sys.argv[1])
    # prefill: from the first embedding widen (k_f32_to_f64); decode steps start at the greedy
    # argmax + embed kernel (k_greedy_next) or, teacher-forced, at the later widens
    widen = [i for i, s in enumerate(seq) if "k_f32_to_f64" in s[0]]
    greedy = [i for i, s in enumerate(seq) if "k_greedy_next" in s[0]]
    if widen:
        steps = greedy if greedy else widen[1:]
        steps = [i for i in steps if i > widen[0]]
        summarize(seq[widen[0]:steps[0]] if steps else seq[widen[0]:], "prefill")
        if steps:
            summarize(seq[steps[0]:steps[1]] if len(steps) > 1 else seq[steps[0]:], "decode step")
    else:
        summarize(seq, "all")
