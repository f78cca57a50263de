"""Generates tests/golden/simulate_golden.json: reports of the reference's OWN
public C ABI (uspsim_run, include/uspsim.h) for the requests below, from
oracle/_ref/libuspsim_api.so (oracle/Makefile target `api`, compiled from
/root/reference/proj/src; nothing copied). Run here, where /root/reference
exists:  make -C oracle api && python tests/golden/make_simulate_golden.py

The B200 `uspsim_run` (include/usp_sim.h) is compared with these reports by
tests/test_simulate.py: invalid-input reports byte for byte, simulate reports
field by field (mesh, shape, ledger minus the position all_gathers)."""
import ctypes
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "..", "..", "oracle", "_ref", "libuspsim_api.so")

# invalid inputs: every rejection path of cmd_simulate / run_command
INVALID = [
    {"command": "simulate", "params": {"seqlen": 64, "ulysses": 16}},
    {"command": "simulate", "params": {"seqlen": 63, "ring": 2, "causal": True}},
    {"command": "simulate", "params": {"seqlen": 64, "ring": 3}},
    {"command": "simulate", "params": {"seqlen": 12, "ring": 2, "ulysses": 4, "kv_heads": 4, "heads": 8}},
    {"command": "simulate", "params": {"heads": 6, "kv_heads": 4}},
    {"command": "simulate", "params": {"seqlen": 0}},
    {"command": "simulate", "params": {"head_size": -3}},
    {"command": "simulate", "params": {"ulysses": 0}},
    {"command": "simulate", "params": {"ring": -1}},
    {"command": "simulate", "params": {"seqlen": "a"}},
    {"command": "simulate", "params": {"causal": 1}},
    {"command": "simulate", "params": 5},
    {"params": {}},
    {"command": "foo"},
    {"command": "simulate", "params": {"seqlen": 63, "ring": 2, "causal": True, "tolerance": 1e-05, "x": 0.1,
                                       "y": 1e16, "z": 123.456, "w": -0.0, "big": 18446744073709551615,
                                       "neg": -7, "s": "a\"b\\c\né", "arr": [1, 2.5, None, True]}},
]
# the balance command (zigzag vs contiguous causal load), host-only
BALANCE = [
    {"command": "balance", "params": {}},
    {"command": "balance", "params": {"seqlen": 64, "ring": 4}},
    {"command": "balance", "params": {"seqlen": 131072, "ring": 8}},
    {"command": "balance", "params": {"seqlen": 48, "ring": 3}},
    {"command": "balance", "params": {"seqlen": 20, "ring": 4}},
    {"command": "balance", "params": {"seqlen": 16, "ring": 0}},
    {"command": "balance", "params": {"seqlen": 12, "ring": 1}},
]
# runnable simulations (the B200 side runs them in bf16; compared on structure + ledger)
SIMULATE = [
    {"command": "simulate", "params": {"seqlen": 64, "heads": 8, "kv_heads": 2, "head_size": 16, "ulysses": 2,
                                       "ring": 2, "causal": True, "check": True}},
    {"command": "simulate", "params": {"seqlen": 256, "heads": 8, "kv_heads": 8, "head_size": 64, "ulysses": 1,
                                       "ring": 4, "causal": True, "check": True, "seed": 3}},
    {"command": "simulate", "params": {"seqlen": 128, "heads": 8, "kv_heads": 4, "head_size": 32, "ulysses": 4,
                                       "ring": 1, "causal": False, "check": True, "batch": 2}},
    {"command": "simulate", "params": {"seqlen": 96, "heads": 4, "kv_heads": 2, "head_size": 128, "ulysses": 1,
                                       "ring": 1, "causal": True, "check": True}},
    {"command": "simulate", "params": {"seqlen": 128, "heads": 8, "kv_heads": 2, "head_size": 64, "ulysses": 2,
                                       "ring": 4, "causal": True, "check": False, "seed": 9}},
]


def main():
    lib = ctypes.CDLL(LIB)
    lib.uspsim_run.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
    for f in ("uspsim_report_json", "uspsim_report_text", "uspsim_report_ledger_csv"):
        getattr(lib, f).restype = ctypes.c_char_p
        getattr(lib, f).argtypes = [ctypes.c_void_p]
    lib.uspsim_report_free.argtypes = [ctypes.c_void_p]
    lib.uspsim_last_error.restype = ctypes.c_char_p

    def run(req):
        text = req if isinstance(req, str) else json.dumps(req)
        h = ctypes.c_void_p()
        st = lib.uspsim_run(text.encode(), ctypes.byref(h))
        if not h.value:
            return {"request": text, "status": st, "json": None, "text": lib.uspsim_last_error().decode(), "csv": ""}
        out = {"request": text, "status": st, "json": lib.uspsim_report_json(h).decode(),
               "text": lib.uspsim_report_text(h).decode(), "csv": lib.uspsim_report_ledger_csv(h).decode()}
        lib.uspsim_report_free(h)
        return out

    golden = {"invalid": [run(r) for r in INVALID] + [run("xx"), run("{\"command\": }")],
              "balance": [run(r) for r in BALANCE],
              "simulate": [run(r) for r in SIMULATE]}
    with open(os.path.join(HERE, "simulate_golden.json"), "w") as f:
        json.dump(golden, f, indent=1)
    print("wrote", len(golden["invalid"]), "invalid and", len(golden["simulate"]), "simulate reports")


if __name__ == "__main__":
    main()
