#!/usr/bin/env python
"""Benchmark of the B200 state-vector gate engine (BASELINE.json metric, configs[1] + configs[2]).

One STEP = the 1q sweep (one Haar U2 on every target 0..29) followed by the 2q sweep (CNOT, CPhase,
Haar U4 on the 21 pairs of {0,1,5,12,20,28,29}) on a 30-qubit (16 GiB) state per GPU, each gate a
separate qs_apply_* call = one single-op kernel (the per-gate GB/s the metric names).
value = algorithmic bytes of all gates of the step on all GPUs / step time (max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-circuits]

N > 1: one process per GPU.  Under torchrun (WORLD_SIZE set) it must equal N; without it bench.py
launches `torch.distributed.run --nproc-per-node N` on itself, and exits non-zero when the node has
fewer than N GPUs (it never prints an N=1 line for N > 1).  Shard = 2^30 amplitudes per GPU (weak
scaling), every sweep gate is on a local qubit.  Extra N > 1 legs: "global" (SURVEY.md §8(d) config 6:
a Haar U2 on every global qubit and a SWAP(local, global) of an n = 32 state, plus n = 34 / 35 at
N = 8 — GB/s per direction and fraction of 900 GB/s, buffered NCCL exchange and CUDA-IPC peer kernels),
"nccl_cal" (the "Cal" row: pairwise NCCL send/recv of 8 GiB), "global_single_process_peer" (the NCCL-free
NVLink path: rank 0 drives every GPU through one handle, fused peer-memory kernels), and the circuits
sharded (strong scaling at n = 32; RQC(34) and QFT(35) at N = 8).
--impl reference: the oracle (plain CPU C code, oracle/) on the host cores, a fixed sample of the step.
--oracle-sweep: the SURVEY.md §8(d) CPU-baseline records (every target t = 0..29 with 1 warm-up + 3
reps, the config-3 pairs, 1-thread rates at t in {0, 15, 29}); --oracle-circuits: the circuit records.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from qsinputs import circuits as C  # noqa: E402

N_LOCAL = 30
# host cores available to this process, read before the oracle's OpenMP runtime pins the main thread
HOST_CORES = len(os.sched_getaffinity(0))
METRIC = "1q/2q gate HBM GB/s (configs[1]+[2] sweeps, n=30/GPU, algorithmic bytes)"


def gate_bytes(g, m):
    """Algorithmic bytes (read + write of the amplitudes the gate must modify)."""
    amps = 1 << m
    if g.kind == "1q":
        return 32 * amps
    if g.kind == "2q":
        return 32 * amps
    if g.name == "CPhase":
        return 8 * amps
    return 16 * amps  # CNOT / general controlled: half the amplitudes


def gate_bytes_sector(g, m):
    """Sector-effective bytes: a 32-B DRAM sector holds the amplitude pair (2j, 2j+1),
    so a gate that selects amplitudes by qubit 0 (control or phase bit) still moves whole sectors."""
    b = gate_bytes(g, m)
    if g.kind == "c1q" and g.q0 == 0:
        return 2 * b
    return b


def gate_bytes_atom(g, m):
    """Atom-effective bytes: the DRAM reads whole 64-B atoms (amplitudes 4j..4j+3, qubits 0 and 1) and
    writes 32-B sectors (pairs 2j, 2j+1).  A gate that touches only the amplitudes whose selecting qubits
    (controls / phase bits) have given values reads every 64-B atom holding one of them and writes every
    sector holding one: bytes = 16 * 2^m * (2^-|S minus {0,1}| + 2^-|S minus {0}|), S = the selecting qubits.
    Measured in round 2 (profiles/r02_granule.txt): cudaLimitMaxL2FetchGranularity = 32 changes neither
    the time nor the DRAM bytes of CNOT(1, x) / CPhase(1, x), so the 64-B read atom is physical."""
    if g.kind in ("1q", "2q"):
        return 32 << m
    sel = {g.q0} if g.name != "CPhase" else {g.q0, g.q1}  # CNOT / controlled U: control; CPhase: both bits
    rd = 2.0 ** -len(sel - {0, 1})
    wr = 2.0 ** -len(sel - {0})
    return int((16 << m) * (rd + wr))


def workload():
    return C.sweep_1q(N_LOCAL) + C.sweep_2q()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, nm in enumerate(names):
                if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy_)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as f:
            return json.load(f).get("dominant_traffic_bytes")
    except Exception:
        return None


# ------------------------------------------------------------------------------------------------
# oracle (CPU) sample: cpu_baseline and --impl reference
# ------------------------------------------------------------------------------------------------
ORACLE_SAMPLE = (("1q", 0), ("1q", 15), ("1q", 29), ("2q", (0, 1)), ("2q", (12, 20)), ("2q", (28, 29)))


def oracle_env():
    """The oracle's OpenMP placement: recorded in every CPU record, set before liborc.so loads."""
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = None
    return {"cpu_model": model, "OMP_PROC_BIND": os.environ["OMP_PROC_BIND"], "OMP_PLACES": os.environ["OMP_PLACES"],
            "OMP_NUM_THREADS": os.environ.get("OMP_NUM_THREADS")}


def _oracle_gates(n):
    """A FIXED sample of the step (no time budget, so every run times the same gates): the Haar U2 on
    t in {0, 15, 29} and CNOT / CPhase / Haar U4 on the pairs (0,1), (12,20), (28,29)."""
    wl = workload()
    out = []
    for kind, q in ORACLE_SAMPLE:
        if kind == "1q":
            out += [g for g in wl if g.kind == "1q" and g.q0 == q]
        else:
            out += [g for g in wl if g.kind != "1q" and (g.q0, g.q1) == q]
    return [g for g in out if max(g.qubits()) < n]


def oracle_sample(reps=3):
    """The oracle (OpenMP over the host cores) on the fixed sample at n = 30 (n = 28 when the host cannot
    hold 16 GiB): 1 untimed warm-up + `reps` timed applications of each gate, min per gate (the paper's
    protocol).  Returns (GB/s, seconds of the mins, description, threads, env)."""
    import psutil
    env = oracle_env()
    from oracle import Oracle
    orc = Oracle()
    n = N_LOCAL if psutil.virtual_memory().available > 24 * 2 ** 30 else 28
    n = int(os.environ.get("QS_ORACLE_N", n))  # (CPU tests of the launch plumbing use a small state)
    a = np.zeros(1 << n, dtype=np.complex128)  # every page touched before timing
    a[0] = 1.0  # the oracle's cost does not depend on the values
    byt, secs = 0, 0.0
    for g in _oracle_gates(n):
        ts = []
        for r in range(reps + 1):
            t = time.perf_counter()
            orc.run(a, [g])
            if r:
                ts.append(time.perf_counter() - t)
        secs += min(ts)
        byt += gate_bytes(g, n)
    cores = int(os.environ.get("OMP_NUM_THREADS", HOST_CORES))
    desc = (f"oracle (C, OpenMP, {cores} threads) at n={n}, fixed sample of the step: Haar U2 on t=0,15,29 and "
            f"CNOT/CPhase/Haar U4 on (0,1),(12,20),(28,29); 1 warm-up + {reps} reps, min per gate")
    return byt / secs / 1e9, secs, desc, cores, env


def oracle_one_thread(ts=(0, 15, 29), n=N_LOCAL):
    """1-thread oracle rate of the Haar U2 at the given targets, in a subprocess with
    OMP_NUM_THREADS=1 (libgomp reads it once per process)."""
    import subprocess as sp
    env = dict(os.environ, OMP_NUM_THREADS="1")
    code = ("import sys, time, json, numpy as np; sys.path.insert(0, %r); from oracle import Oracle; "
            "from qsinputs import circuits as C; o = Oracle(); a = np.zeros(1 << %d, dtype=np.complex128); a[0] = 1; "
            "out = {}\nfor t in %r:\n    g = C.sweep_1q(30)[t]; t0 = time.perf_counter(); o.run(a, [g]); "
            "out[t] = (32 << %d) / (time.perf_counter() - t0) / 1e9\nprint(json.dumps(out))" % (ROOT, n, tuple(ts), n))
    try:
        r = sp.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        return {f"t{k}": v for k, v in json.loads(r.stdout.strip().splitlines()[-1]).items()}
    except Exception as e:
        return {"error": str(e)[:200]}


def oracle_sweep(out_path):
    """SURVEY.md §8(d) CPU baseline in full: the oracle on every target t = 0..29 of configs[1] (1 warm-up +
    3 reps, min), each configs[2] gate once, and the 1-thread U2 rate at t in {0, 15, 29}; one JSON line per
    record (host cores, CPU model, OMP placement).  A measurement mode, not part of the default bench run."""
    import psutil
    env = oracle_env()
    from oracle import Oracle
    orc = Oracle()
    n = N_LOCAL if psutil.virtual_memory().available > 24 * 2 ** 30 else 28
    cores = int(os.environ.get("OMP_NUM_THREADS", HOST_CORES))
    a = np.zeros(1 << n, dtype=np.complex128)
    a[0] = 1.0
    recs = []
    for g in C.sweep_1q(n):
        ts = []
        for r in range(4):
            t = time.perf_counter()
            orc.run(a, [g])
            if r:
                ts.append(time.perf_counter() - t)
        recs.append({"record": "oracle_gate", "config": "configs[1]", "gate": "U2", "qubits": [g.q0], "n": n,
                     "reps": 3, "t_min_s": min(ts), "t_med_s": statistics.median(ts),
                     "GBps": gate_bytes(g, n) / min(ts) / 1e9, "host_cores": cores, **env})
    for g in C.sweep_2q():
        t = time.perf_counter()
        orc.run(a, [g])
        dt = time.perf_counter() - t
        recs.append({"record": "oracle_gate", "config": "configs[2]", "gate": g.name, "qubits": list(g.qubits()),
                     "n": n, "reps": 1, "t_min_s": dt, "GBps": gate_bytes(g, n) / dt / 1e9, "host_cores": cores, **env})
    recs.append({"record": "oracle_1thread_u2", "n": n, "GBps": oracle_one_thread(n=n), "host_cores": 1, **env})
    with open(out_path, "w") as f:
        for r in recs:
            f.write(json.dumps(r) + "\n")
    u2 = [r["GBps"] for r in recs if r.get("gate") == "U2"]
    print(json.dumps({"records": len(recs), "u2_GBps_min": min(u2), "u2_GBps_max": max(u2), "out": out_path}))


def oracle_circuits():
    """The oracle baseline on circuits (reported only): QFT(28)|x> and grid RQC(25) in
    full on the host cores (OpenMP), the 1-thread rate of a U2 at t in {0, 14, 27} (n = 28), the n = 32
    times extrapolated x16 per 4 qubits (labelled as such), and the GPU on the same circuits.  One JSON
    line per record."""
    import subprocess as sp

    import torch

    import paper_2506_09198_b200 as qs
    from oracle import Oracle
    orc = Oracle()
    cores = int(os.environ.get("OMP_NUM_THREADS", HOST_CORES))
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        model = None
    recs = []
    for name, n, circ, init in (("QFT|x>", 28, C.qft(28), C.qft_x(28)), ("grid RQC", 25, C.rqc_grid(25), 0)):
        a = orc.basis(n, init)
        t0 = time.perf_counter()
        orc.run(a, circ)
        t_cpu = time.perf_counter() - t0
        ref = a
        with qs.QState(n) as st:
            st.set_option("jit_async", 0)
            ss = torch.cuda.ExternalStream(st.stream(0))
            ts = []
            for r in range(4):
                st.init_basis(init)
                st.sync()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(ss)
                st.run(circ)
                e1.record(ss)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1) / 1e3)
            got = st.read()
        recs.append({"record": "oracle_circuit", "circuit": name, "n": n, "gates": len(circ), "oracle_s": t_cpu,
                     "host_cores": cores, "cpu_model": model, "gpu_s": min(ts[1:]),
                     "gpu_vs_oracle": t_cpu / min(ts[1:]), "max_abs_diff": float(np.max(np.abs(got - ref))),
                     "oracle_s_n32_extrapolated": t_cpu * 16 ** ((32 - n) / 4) * (len(C.qft(32) if "QFT" in name else
                                                                                       C.rqc_grid(32)) / len(circ)),
                     "extrapolation": "x16 per 4 qubits and x(gates at n=32 / gates here): extrapolated, not measured"})
    n = 28
    for t in (0, 14, 27):
        env = dict(os.environ, OMP_NUM_THREADS="1")
        code = ("import sys, time, numpy as np; sys.path.insert(0, %r); from oracle import Oracle; "
                "from qsinputs import circuits as C; o = Oracle(); a = o.random_state(%d, 2506); "
                "g = C.sweep_1q(30)[%d]; t0 = time.perf_counter(); o.run(a, [g]); print(time.perf_counter() - t0)"
                % (os.path.dirname(os.path.abspath(__file__)), n, t))
        r = sp.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        secs = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None
        recs.append({"record": "oracle_1thread_u2", "n": n, "t": t, "oracle_s": secs, "host_cores": 1,
                     "GBps": (32 << n) / secs / 1e9 if secs else None})
    for r in recs:
        print(json.dumps(r), flush=True)


def run_reference(args, rank, world):
    if rank != 0:
        return
    K, W = args.steps, args.warmup
    vals = []
    for i in range(W + K):
        gbs, secs, desc, cores, env = oracle_sample(reps=1)  # one application of each sample gate per step
        if i >= W:
            vals.append((gbs, secs))
    v = statistics.median(x[0] for x in vals)
    ms = statistics.median(x[1] for x in vals) * 1e3
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "configs[1]+configs[2] sweeps (bounded oracle sample per step)", "n_qubits": N_LOCAL},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": cores, "kind": "oracle",
                             "sample": desc, **env},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-circuits", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ipc", action="store_true", help="N > 1: also time global-qubit gates over the CUDA-IPC "
                                                        "peer-memory transport (QS_P2P_RANK=1)")
    ap.add_argument("--no-sp", action="store_true", help="N > 1: skip the single-process peer-memory leg")
    ap.add_argument("--oracle-circuits", action="store_true",
                    help="SURVEY.md §8(d) CPU-baseline records instead of the bench line: the oracle on QFT(28) and "
                         "grid RQC(25) in full, its 1-thread U2 rate, the GPU on the same circuits")
    ap.add_argument("--oracle-sweep", default=None, metavar="OUT.jsonl",
                    help="SURVEY.md §8(d) CPU-baseline records of the full sweep instead of the bench line")
    args = ap.parse_args()
    if args.oracle_circuits:
        return oracle_circuits()
    if args.oracle_sweep:
        return oracle_sweep(args.oracle_sweep)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        return launch_ranks(args.gpus)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2506_09198_b200 as qs

    if torch.cuda.device_count() <= local_rank:
        print(f"bench.py: rank {rank} needs GPU {local_rank}, the node has {torch.cuda.device_count()}", file=sys.stderr)
        sys.exit(1)
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        # communicator init lines (ranks, devices, transports) for the record — on stderr, so that stdout
        # carries rank 0's JSON line only, whatever order the ranks' communicators are torn down in
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        assert dist.get_world_size() == args.gpus
    k = world.bit_length() - 1
    n = N_LOCAL + k
    if world > 1:
        obj = [qs.qs_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        st = qs.QState.rank(n, world, rank, local_rank, obj[0])
    else:
        st = qs.QState(n)
    m = st.info["m"]
    st.init_random(2506)
    stream = torch.cuda.ExternalStream(st.stream(0))
    wl = workload()
    step_bytes = sum(gate_bytes(g, m) for g in wl)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        st.sync()

    def one_step(events=None):
        for i, g in enumerate(wl):
            if events is not None:
                events[i][0].record(stream)
            st.apply(g)
            if events is not None:
                events[i][1].record(stream)

    for _ in range(args.warmup):
        one_step()
    barrier()
    K = args.steps
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in wl] for _ in range(K)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = st.launches()
    with Clocks(local_rank) as clk:
        barrier()
        start.record(stream)
        for s in range(K):
            one_step(evs[s])
        stop.record(stream)
        barrier()
    launches = st.launches() - l0
    total_ms = start.elapsed_time(stop)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / K
    value = step_bytes * world / (ms_per_step / 1e3) / 1e9

    # per-kernel durations (the dominant kernels: general U2 pair and U4 quad)
    per = {}
    for i, g in enumerate(wl):
        key = {"1q": "U2", "2q": "U4"}.get(g.kind, g.name)
        ds = [evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(K)]
        per.setdefault(key, []).append((g, statistics.median(ds)))
    peak, peak_src = measured_peak()
    kernels = {}
    for key, lst in per.items():
        tot_b = sum(gate_bytes(g, m) for g, _ in lst)
        tot_ms = sum(d for _, d in lst)
        tot_e = sum(gate_bytes_sector(g, m) for g, _ in lst)
        tot_a = sum(gate_bytes_atom(g, m) for g, _ in lst)
        kernels[key] = {"launches_per_step": len(lst), "avg_ms": tot_ms / len(lst),
                        "gbs": tot_b / (tot_ms / 1e3) / 1e9, "frac_of_peak": tot_b / (tot_ms / 1e3) / 1e9 / peak,
                        "sector_gbs": tot_e / (tot_ms / 1e3) / 1e9, "atom_eff_gbs": tot_a / (tot_ms / 1e3) / 1e9,
                        "atom_eff_frac_of_peak": tot_a / (tot_ms / 1e3) / 1e9 / peak}
    per_target = [{"t": g.q0, "ms": d, "gbs": gate_bytes(g, m) / (d / 1e3) / 1e9} for g, d in per["U2"]]
    # [gate, q0, q1, ms, algorithmic GB/s, atom-effective GB/s (64-B read atoms, 32-B write sectors)]
    per_gate_2q = [[g.name, g.q0, g.q1, round(d, 4), round(gate_bytes(g, m) / (d / 1e3) / 1e9, 1),
                    round(gate_bytes_atom(g, m) / (d / 1e3) / 1e9, 1)]
                   for key in ("CNOT", "CPhase", "U4") for g, d in per.get(key, [])]
    u2 = kernels["U2"]
    share = sum(d for _, d in per["U2"]) / ms_per_step
    roofline = {"bound": "hbm", "achieved": u2["gbs"], "peak": peak, "unit": "GB/s", "frac": u2["gbs"] / peak,
                "traffic": ncu_traffic(), "kernel": "k_pair (general 1q U2, t=0..29)",
                "alg_bytes_per_launch": 32 * (1 << m), "avg_launch_ms": u2["avg_ms"], "share_of_step": share,
                "peak_source": peak_src}
    try:  # a second, live ceiling with the gate kernels' access pattern: in-place read-modify-write
        ip = inplace_ceiling(torch)
        roofline.update({"ceiling_inplace_gbs": ip, "frac_of_inplace": u2["gbs"] / ip,
                         "ceiling_inplace_note": "torch in-place mul_ over 16 GiB fp64, read + write bytes, best of 5, "
                                                 "measured in this run (the peak above is the driver's copy_ figure)"})
    except Exception as e:  # report, do not hide
        roofline["ceiling_inplace_error"] = str(e)[:200]

    # e2e through the public API with host buffers (pinned), copies inside the timed region: every
    # step copies its full input state host -> device (qs_write_amps_async), runs the step's gates
    # (qs_apply_*) and copies its result state device -> host (qs_read_amps_async).  Steps rotate over
    # E handles (one stream each), so one step's copies overlap another step's gates (copy engines and
    # SMs busy at once), the way a serving loop would pipeline independent jobs.
    e2e = None
    if not args.no_e2e:
        try:
            e2e = bench_e2e(qs, torch, st, wl, n, m, rank, world, local_rank, dist, barrier, step_bytes)
        except Exception as e:  # report, do not hide (e.g. host memory exhausted)
            e2e = {"value": None, "unit": "GB/s", "error": str(e)[:300]}

    st.close()
    # global-qubit gates over NVLink and the NCCL send/recv ceiling (N > 1, Cal)
    glob = cal = None
    if world > 1:
        cal = bench_nccl_cal(torch, dist, rank, world)
        glob = bench_global(qs, torch, dist, rank, world, local_rank, transport="nccl")
    vglob = bench_virtual_global(qs, torch) if world == 1 and not args.no_circuits else None
    circuits = None
    if not args.no_circuits:
        circuits = bench_circuits(qs, torch, world, rank, local_rank, dist)
    glob_sp = None
    if world > 1 and not args.no_sp:  # the NCCL-free NVLink path: one process driving every GPU of the node
        glob_sp = bench_single_process_peer(qs, torch, dist, rank, world)
    if world > 1 and args.ipc:  # last, opt-in: the CUDA-IPC peer-memory transport (QS_P2P_RANK=1), which
        # no run has executed yet (this pool has one GPU per box); a failure there must not cost the line
        glob_ipc = bench_global(qs, torch, dist, rank, world, local_rank, transport="ipc")
        glob = {"nccl": glob, "ipc": glob_ipc}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gbs, secs, desc, cores, env = oracle_sample()
        cpu = {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "oracle", "sample": desc, "seconds": secs,
               **env, "one_thread_gbs_n30": oracle_one_thread()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": "configs[1]+configs[2]: Haar U2 on t=0..29, then CNOT/CPhase/Haar U4 on the 21 pairs "
                           "of {0,1,5,12,20,28,29}; one qs_apply_* (one kernel) per gate",
                           "n_qubits": n, "local_qubits": m, "gates_per_step": len(wl), "alg_bytes_per_step": step_bytes * world,
                           "l2": "inputs larger than L2 (16 GiB state per GPU vs 126 MB L2); no flush",
                           "parallelism": f"state sharded on top {k} qubits" if k else "single GPU"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "kernels": kernels, "u2_per_target": per_target,
                "per_gate_2q": per_gate_2q}
        if glob:
            line["global"] = glob
        if glob_sp:
            line["global_single_process_peer"] = glob_sp
        if cal:
            line["nccl_cal"] = cal
        if vglob:
            line["global_virtual_1gpu"] = vglob
        if circuits:
            line["circuits"] = circuits
    if dist:
        dist.destroy_process_group()
    if rank == 0:  # last, after every communicator is gone (NCCL's INFO lines come before it)
        print(json.dumps(line), flush=True)


def bench_nccl_cal(torch, dist, rank, world, nbytes=8 << 30, reps=3):
    """SURVEY.md §8(d) "Cal": pairwise NCCL send/recv of 8 GiB per direction between rank pairs (partner
    rank ^ 1, and rank ^ N/2 for N >= 4) — the NVLink ceiling the global-gate numbers are read against.
    CUDA events on the current stream (the work handles make it wait for NCCL), max over ranks."""
    out = {}
    try:
        send = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
        recv = torch.empty_like(send)
        for name, partner in (("xor1", rank ^ 1), ("xor_half", rank ^ (world // 2))):
            if name == "xor_half" and world < 4:
                continue

            def once():
                for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, send, partner),
                                                 dist.P2POp(dist.irecv, recv, partner)]):
                    r.wait()
            once()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                once()
            b.record()
            b.synchronize()
            t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            out[name] = {"bytes_per_direction": nbytes, "ms": ms, "gbs_per_direction": nbytes / ms / 1e6,
                         "frac_of_900": nbytes / ms / 1e6 / 900.0}
        del send, recv
        torch.cuda.empty_cache()
    except Exception as e:  # report, do not hide
        out["error"] = str(e)[:300]
    return out


def bench_global(qs, torch, dist, rank, world, local_rank, transport="nccl", reps=3):
    """SURVEY.md §8(d) config 6 (the north star's NVLink bar): a Haar U2 on every global qubit and a
    SWAP(top local qubit, global qubit) of an n = 32 state sharded over the N ranks (and n = 34 / 35 at
    N = 8), one process per GPU.  transport "nccl": the chunked, double-buffered ncclSend/ncclRecv
    exchange fused with the update; "ipc": the CUDA-IPC peer-memory kernels (QS_P2P_RANK=1).  GB/s per
    direction = 16 * 2^m / t (U2) or 8 * 2^m / t (SWAP), against 900 GB/s; device time, max over ranks."""
    recs = []
    k = world.bit_length() - 1
    U = C.sweep_1q(1)[0].m
    SW = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
    prev = os.environ.get("QS_P2P_RANK")
    os.environ["QS_P2P_RANK"] = "1" if transport == "ipc" else "0"
    try:
        for n in [32] + ([34, 35] if world == 8 else []):
            m = n - k
            obj = [qs.qs_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            with qs.QState.rank(n, world, rank, local_rank, obj[0]) as st:
                st.init_random(2506)
                ss = torch.cuda.ExternalStream(st.stream(0))
                gates = [("U2", g, C.g1(g, U), 16 << m) for g in range(m, n)] + \
                        [("SWAP", g, C.g2(m - 1, g, SW), 8 << m) for g in range(m, n)]
                for name, g, gate, nvb in gates:
                    st.apply(gate)
                    st.sync()
                    dist.barrier()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(ss)
                    for _ in range(reps):
                        st.apply(gate)
                    b.record(ss)
                    st.sync()
                    t = torch.tensor([a.elapsed_time(b) / reps], device="cuda")
                    dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    ms = float(t.item())
                    bar = nvb / (0.7 * 900e9) * 1e3
                    recs.append({"n": n, "P": world, "gate": name, "global_qubit": g, "ms": round(ms, 4),
                                 "nvlink_bytes_per_direction": nvb, "gbs_per_direction": round(nvb / ms / 1e6, 1),
                                 "frac_of_900": round(nvb / ms / 1e6 / 900.0, 4), "bar_70pct_ms": round(bar, 3)})
                assert abs(1 - st.norm2()) <= 1e-12
    except Exception as e:  # report, do not hide
        recs.append({"error": str(e)[:300]})
    finally:
        if prev is None:
            os.environ.pop("QS_P2P_RANK", None)
        else:
            os.environ["QS_P2P_RANK"] = prev
    return {"transport": transport, "records": recs}


def bench_single_process_peer(qs, torch, dist, rank, world, n=32, reps=3):
    """SURVEY.md §8(f) rank 3, the NCCL-free NVLink path: rank 0 alone drives all N GPUs of the node through
    ONE handle (qs_create(n, N): peer access between every pair), so a global-qubit gate is ONE fused
    peer-memory kernel per device — each loads its own and its partner's amplitude over NVLink, applies the
    gate and stores both (k_p2p.cu) — with no exchange buffer and no NCCL.  A Haar U2 on every global qubit
    and a SWAP(top local, global) of an n = 32 state; per gate the max over devices of the device time (CUDA
    events on each device's library stream); GB/s per direction = 16 * 2^m / t (U2), 8 * 2^m / t (SWAP).
    The other ranks wait at a CPU (gloo) barrier, so no kernel of theirs runs meanwhile."""
    cpu_pg = dist.new_group(backend="gloo")
    dist.barrier(group=cpu_pg)
    out = None
    if rank == 0:
        recs = []
        try:
            k = world.bit_length() - 1
            m = n - k
            U = C.sweep_1q(1)[0].m
            SW = np.eye(4, dtype=np.complex128)[[0, 2, 1, 3]]
            with qs.QState(n, world) as st:
                st.init_random(2506)
                streams = [torch.cuda.ExternalStream(st.stream(i), device=i) for i in range(world)]
                gates = [("U2", g, C.g1(g, U), 16 << m) for g in range(m, n)] + \
                        [("SWAP", g, C.g2(m - 1, g, SW), 8 << m) for g in range(m, n)]
                for name, g, gate, nvb in gates:
                    st.apply(gate)
                    st.sync()
                    ev = []
                    for i in range(world):
                        with torch.cuda.device(i):
                            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                            a.record(streams[i])
                        ev.append((a, b))
                    for _ in range(reps):
                        st.apply(gate)
                    for i in range(world):
                        with torch.cuda.device(i):
                            ev[i][1].record(streams[i])
                    st.sync()
                    ms = max(a.elapsed_time(b) for a, b in ev) / reps
                    recs.append({"n": n, "P": world, "gate": name, "global_qubit": g, "ms": round(ms, 4),
                                 "nvlink_bytes_per_direction": nvb, "gbs_per_direction": round(nvb / ms / 1e6, 1),
                                 "frac_of_900": round(nvb / ms / 1e6 / 900.0, 4)})
                recs.append({"norm_err": abs(1 - st.norm2())})
        except Exception as e:  # report, do not hide
            recs.append({"error": str(e)[:300]})
        out = {"transport": "single-process peer memory (qs_create(n, N), k_p2p.cu)", "records": recs}
    dist.barrier(group=cpu_pg)
    return out


def launch_ranks(n_gpus):
    """--gpus N without torchrun: run this script under torch.distributed.run with N processes, one per
    GPU.  A node with fewer than N GPUs is an error (exit 1), never a silent N=1 measurement."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < n_gpus:
        print(f"bench.py: --gpus {n_gpus} needs {n_gpus} GPUs, this node has {have}", file=sys.stderr)
        sys.exit(1)
    with socket.socket() as sk:  # a free rendezvous port on the loopback interface
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n_gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def bench_e2e(qs, torch, st, wl, n, m, rank, world, local_rank, dist, barrier, step_bytes):
    """e2e through the public API with host buffers (pinned), copies inside the timed region: every step
    copies its full input shard host -> device (qs_write_amps_async), runs the step's gates (qs_apply_*)
    and copies its result shard device -> host (qs_read_amps_async).  Steps rotate over E handles (one
    stream each), so one step's copies overlap another step's gates (copy engines and SMs busy at once),
    the way a serving loop pipelines independent jobs.  E is bounded by the host RAM the node's ranks
    share (one pinned shard-sized buffer per handle)."""
    import psutil
    shard = 16 << m
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    budget = 0.5 * psutil.virtual_memory().available / max(1, local_world)
    E = min(int(os.environ.get("QS_E2E_HANDLES", "4")), int(budget // shard))
    if E < 1:
        return {"value": None, "unit": "GB/s",
                "unavailable": f"host RAM: {local_world} ranks x {shard / 2**30:.0f} GiB pinned shard buffers exceed "
                               f"half of the {psutil.virtual_memory().available / 2**30:.0f} GiB available"}
    handles = [st]
    extra = []
    for _ in range(E - 1):
        if world > 1:
            obj = [qs.qs_get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            h = qs.QState.rank(n, world, rank, local_rank, obj[0])
        else:
            h = qs.QState(n)
        handles.append(h)
        extra.append(h)
    try:
        hosts = []
        for _ in range(E):
            hb = torch.empty((1 << m) * 2, dtype=torch.float64, pin_memory=True).numpy().view(np.complex128)
            qs.qs_read_amps(st.h, rank << m, 1 << m, hb)
            hosts.append(hb)
        Ke = int(os.environ.get("QS_E2E_STEPS", str(12 * E)))  # the pipeline fill (first upload) and drain
        # (last download, ~0.3 s each at PCIe rate) amortise over 12E steps (~4 % of the wall clock)
        for h in handles:
            h.sync()
        # the host link's duplex ceiling, measured here: one shard up (into handle 1) while another comes
        # down (from handle 0), no gates — the copies a step needs, at full link speed; every host buffer
        # still holds the step input afterwards (handle 0's state is that input)
        link = None
        if E >= 2:
            tl = time.perf_counter()
            qs.qs_write_amps_async(handles[1].h, rank << m, hosts[0])
            qs.qs_read_amps_async(handles[0].h, rank << m, 1 << m, hosts[1])
            handles[0].sync()
            handles[1].sync()
            link = shard / (time.perf_counter() - tl) / 1e9
        barrier()
        streams = [torch.cuda.ExternalStream(h.stream(0)) for h in handles]
        t0 = time.perf_counter()
        prev = None
        for sidx in range(Ke):
            h, hb, hs = handles[sidx % E], hosts[sidx % E], streams[sidx % E]
            qs.qs_write_amps_async(h.h, rank << m, hb)
            if prev is not None:  # the steps' gates run one step at a time (full HBM each); the
                hs.wait_event(prev)  # copies of the other handles proceed underneath them
            for g in wl:
                h.apply(g)
            prev = torch.cuda.Event()
            prev.record(hs)
            qs.qs_read_amps_async(h.h, rank << m, 1 << m, hb)
        for h in handles:
            h.sync()
        barrier()
        e2e_s = (time.perf_counter() - t0) / Ke
        if dist:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        return {"value": step_bytes * world / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": shard,
                "d2h_bytes_per_step": shard, "ms_per_step": e2e_s * 1e3, "steps": Ke, "handles": E,
                # each step moves one shard each way over the host link; when this rate is the link's
                # concurrent-duplex rate the e2e value is bound by PCIe, not by the gates
                "link_gbs_per_direction": shard / e2e_s / 1e9, "link_duplex_ceiling_gbs": link,
                "what": "per step: qs_write_amps_async(full shard from pinned host) + the step's qs_apply_* calls + "
                        "qs_read_amps_async(full shard to pinned host); steps rotate over the handles so copies "
                        "overlap other steps' gates (the gates of consecutive steps are ordered by an event "
                        "on the library stream); wall clock from the first copy to the last sync"}
    finally:
        for h in extra:
            h.close()


def bench_circuits(qs, torch, world=1, rank=0, local_rank=0, dist=None):
    """configs[3]/[4] at n = 32: QFT of |x> and grid RQC, fused — one GPU holds the 64 GiB state, N > 1
    GPUs shard it (strong scaling; one process per GPU, the library's exchanges over NCCL).  Device
    time per run on each rank (CUDA events on the library stream), max over ranks."""
    out = {}
    runs = [("qft_n32", 32, C.qft(32), ("basis", C.qft_x(32))), ("rqc_n32", 32, C.rqc_grid(32), ("basis", 0))]
    if world == 8:  # configs[3] n = 34 and configs[4] n = 35 (512 GiB), sharded over 8 GPUs
        runs += [("rqc_n34", 34, C.rqc_grid(34), ("basis", 0)), ("qft_n35", 35, C.qft(35), ("basis", C.qft_x(35)))]
    for name, n, circ, init in runs:
        try:
            if world > 1:
                obj = [qs.qs_get_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                st = qs.QState.rank(n, world, rank, local_rank, obj[0])
            else:
                st = qs.QState(n)
            with st:
                stream = torch.cuda.ExternalStream(st.stream(0))
                ts = []
                for rep in range(4):
                    if init[0] == "basis":
                        st.init_basis(init[1])
                    st.sync()
                    if dist:
                        dist.barrier()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    st.run(circ)
                    b.record(stream)
                    st.sync()
                    t = a.elapsed_time(b) / 1e3
                    if dist:
                        tt = torch.tensor([t], device="cuda")
                        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                        t = float(tt.item())
                    ts.append(t)
                passes, exch = st.last_plan()
                norm = st.norm2()
                jit = st.jit_stats()
                cold = None
                if name.startswith("rqc"):
                    # a never-seen seed, end to end as the paper times RQC ("including state
                    # initialization, random gate generation"): gate generation + init + planning + any
                    # kernel compilation + the gates, wall clock (max over ranks).  The first seed's run
                    # queued the shape's FAMILY kernels for background compilation (jit_tile.cu); they are
                    # joined first, as a process that has run this circuit shape once would have them
                    st.set_option("jit_wait", 1)
                    c0 = st.jit_stats()["compiled"]
                    if dist:
                        dist.barrier()
                    t0 = time.perf_counter()
                    c2 = C.rqc_grid(n, seed=21)
                    st.init_basis(0)
                    st.run(c2)
                    st.sync()
                    cw = time.perf_counter() - t0
                    if dist:
                        tt = torch.tensor([cw], device="cuda")
                        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                        cw = float(tt.item())
                    jit2 = st.jit_stats()
                    cold = {"cold_seed21_wall_s": cw, "kernels_compiled_for_it": jit2["compiled"] - c0,
                            "cold_what": "never-seen seed 21 of the same circuit shape: rqc_grid generation + init + "
                                         "plan + gates (family pass kernels: sqrtX/sqrtY/sqrtW picked per op at run "
                                         "time), wall clock"}
            fl = _circuit_floor(name) if world == 1 else None
            if fl:  # the circuit's own roofline (FP64 for RQC, HBM for QFT), profiles/r02_fp64_roofline.txt
                fl = dict(fl, frac_of_floor=fl["per_pass_max_floor_s"] / min(ts[1:]),
                          achieved_fp64_ops_per_s=fl["fp64_thread_ops"] / min(ts[1:]))
            out[name] = {"s_min": min(ts[1:]), "s_median": statistics.median(ts[1:]), "gates": len(circ), "roofline": fl,
                         "n_gpus": world, "hbm_passes": passes, "exchange_steps": exch, "norm_err": abs(1 - norm),
                         "pass_gbs_per_gpu": passes * (32 << n) / world / min(ts[1:]) / 1e9,
                         # every HBM pass reads and writes the shard once: its floor at the measured copy rate
                         "pass_floor_s": passes * (32 << n) / world / (_peak_gbs() * 1e9) if _peak_gbs() else None,
                         "model_unfused_s": {"qft_n32": 3.52, "rqc_n32": 15.14}.get(name) if world == 1 else None,
                         "first_run_s": ts[0], "jit_kernels_compiled_total": jit["compiled"], **(cold or {}),
                         "what": "fused tile passes (JIT straight-line kernels); first_run_s includes compiling the pass "
                                 "kernels not yet in the on-disk cache (NVRTC, in parallel)"
                                 + ("; sharded on the top qubits, global-qubit remapping, NCCL exchanges" if world > 1
                                    else "")}
        except Exception as e:  # report, do not hide
            out[name] = {"error": str(e)}
    return out


def inplace_ceiling(torch, nbytes=16 << 30, reps=5):
    """GB/s of torch's in-place x.mul_(c) over nbytes of fp64 (read + write), best of reps."""
    x = torch.ones(nbytes // 8, dtype=torch.float64, device="cuda")
    best = None
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        x.mul_(1.0)
        b.record()
        b.synchronize()
        t = a.elapsed_time(b) / 1e3
        best = t if best is None else min(best, t)
    del x
    torch.cuda.empty_cache()
    return 2 * nbytes / best / 1e9


def bench_virtual_global(qs, torch, n=30, reps=10):
    """One GPU only: a Haar U2 on the global qubit of a state split into 2 virtual shards of the same
    device — the fused peer-memory exchange kernel (k_p2p.cu: each shard reads its own and the partner's
    amplitude, applies the gate, writes both) against the local U2 kernel on the same state.  Every byte
    is local HBM here, so this checks the fused kernel's memory efficiency, NOT NVLink (which needs N > 1)."""
    u = workload()[n - 1].m
    out = {}
    for name, P in (("local_u2_ms", 1), ("virtual_global_u2_ms", 2)):
        with qs.QState(n, P, virtual=P > 1) as st:
            st.init_random(2506)
            ss = torch.cuda.ExternalStream(st.stream(0))
            st.apply_1q(n - 1, u)
            st.sync()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(ss)
            for _ in range(reps):
                st.apply_1q(n - 1, u)
            b.record(ss)
            b.synchronize()
            out[name] = a.elapsed_time(b) / reps
    out["hbm_gbs_virtual_global"] = (32 << n) / (out["virtual_global_u2_ms"] / 1e3) / 1e9
    out["what"] = ("U2 on qubit %d: one shard vs 2 virtual shards of ONE GPU (fused peer-memory exchange kernel); "
                   "local HBM only, not an NVLink number" % (n - 1))
    return out


def _circuit_floor(name):
    """Measured floors of a benchmark circuit (profiles/r02_circuit_floors.json), or None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r02_circuit_floors.json")))
        return dict(d[name], fp64_peak_ops_per_s=d["fp64_peak_ops_per_s"], source="profiles/r02_circuit_floors.json")
    except Exception:
        return None


def _peak_gbs():
    try:
        return float(json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return None


if __name__ == "__main__":
    main()
