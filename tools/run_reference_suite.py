"""Run the reference's own test suite (pyrocell 0.1.0 pkg/tests, staged
in baseline/_ref/pyrocell_tests -- git-ignored, like the reference install)
against this package through the ``pyrocell`` import alias
(tools/pyrocell_alias), on the GPU box:

    python tools/run_reference_suite.py OUT_DIR

Writes OUT_DIR/reference_suite.xml (JUnit) and prints a per-test table."""
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    out = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"))
    os.makedirs(out, exist_ok=True)
    tests = os.path.join(ROOT, "baseline", "_ref", "pyrocell_tests")
    if not os.path.isdir(tests):
        raise SystemExit(f"{tests} missing: stage the reference tests there first")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tools", "pyrocell_alias"), ROOT])
    xml = os.path.join(out, "reference_suite.xml")
    rc = subprocess.call([sys.executable, "-m", "pytest", tests, "-q", "-p", "no:cacheprovider",
                          f"--junitxml={xml}", "-o", "junit_family=xunit1"], env=env, cwd=tests)
    rows = []
    for case in ET.parse(xml).getroot().iter("testcase"):
        name = f"{case.get('file', case.get('classname'))}::{case.get('name')}"
        status, why = "pass", ""
        for tag in ("failure", "error", "skipped"):
            el = case.find(tag)
            if el is not None:
                status = {"failure": "FAIL", "error": "ERROR", "skipped": "skip"}[tag]
                why = (el.get("message") or "").splitlines()[0][:160] if el.get("message") else ""
        rows.append((case.get("classname"), case.get("name"), status, why))
    for r in rows:
        print(" | ".join(r))
    npass = sum(r[2] == "pass" for r in rows)
    print(f"{npass} passed of {len(rows)} (pytest rc {rc})")


if __name__ == "__main__":
    main()
