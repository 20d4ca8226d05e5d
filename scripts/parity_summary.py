"""Summarise a parity record (tests/_harness.RECORD written via $TBA_PARITY_OUT) as a markdown table:
per test / config / seed / quantity, the number of values compared, the max |error| and the max
error / tolerance (1.0 = at the bar). Usage: python scripts/parity_summary.py profiles/parity_r02.json"""
import json
import sys


def main(path):
    d = json.load(open(path))
    recs = d["records"]
    print(f"# GPU parity at full size vs the fp64 oracle ({path})\n")
    print(f"host cores: {d['meta'].get('cores')}, GPU: {d['meta'].get('gpu')}, pytest exit status "
          f"{d['meta'].get('exitstatus')}\n")
    worst = {}
    for r in recs:
        q = r["quantity"].split(" [")[0].split(" (")[0]
        worst[q] = max(worst.get(q, 0.0), r["max_err_over_tol"])
    print("Worst error / tolerance per quantity over every record: " +
          ", ".join(f"{k} {v:.3g}" for k, v in sorted(worst.items())) + "\n")
    print("| test | config | seed | quantity | n | max abs err | max err / tol |")
    print("|---|---|---|---|---|---|---|")
    for r in recs:
        print(f"| {r['test']} | {r['config']} | {r['seed']} | {r['quantity']} | {r['n']} | "
              f"{r['max_abs_err']:.3g} | {r['max_err_over_tol']:.3g} |")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "profiles/parity_r02.json")
