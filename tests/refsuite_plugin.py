"""pytest plugin (test infrastructure): installs the device path into the
reference package before the reference's own test modules import it
(compat.install), and records every test outcome with its failure text into
the JSON file named by GCNB_REFSUITE_OUT.  Used by test_reference_suite.py."""

import json
import os

_results = []


def pytest_configure(config):
    import gcnpart

    from paper_2212_05009_b200 import compat

    compat.install(gcnpart)


def pytest_runtest_logreport(report):
    if report.when == "call" or report.outcome != "passed":
        _results.append({"nodeid": report.nodeid, "when": report.when, "outcome": report.outcome,
                         "longrepr": str(report.longrepr)[-3000:] if report.failed else ""})


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("GCNB_REFSUITE_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(_results, f, indent=1)
