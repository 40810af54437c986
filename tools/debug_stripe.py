import multiprocessing as mp, os, sys, time, secrets, traceback
sys.path.insert(0, os.getcwd())

def helper(ctl_name, j, blob_name, blob_bytes):
    t0 = time.time()
    print(f"[helper {j}] start", flush=True)
    try:
        from paper_2604_26334_b200.runtime import striping
        from paper_2604_26334_b200.runtime import lib as L
        L.lib()
        print(f"[helper {j}] lib loaded {time.time()-t0:.2f}s", flush=True)
        n = striping.helper_main(ctl_name, j, blob_name, blob_bytes)
        print(f"[helper {j}] done copied={n} {time.time()-t0:.2f}s", flush=True)
    except Exception:
        traceback.print_exc()
        sys.stdout.flush()

if __name__ == "__main__":
    import numpy as np
    from paper_2604_26334_b200.planning import catalog
    from paper_2604_26334_b200.planning.graph import total_model_bytes
    from paper_2604_26334_b200.runtime.engine import Engine
    from paper_2604_26334_b200.runtime.striping import StripeLeader
    spec = catalog.builtin_model("tiny-moe")
    budget = 0.9 * total_model_bytes(spec)
    prompt = np.random.default_rng(3).integers(0, spec.vocab_size, 40).astype(np.int32)
    tok = secrets.token_hex(4)
    blob_name, ctl_name = f"pshard_stripe_blob_{tok}", f"pshard_stripe_ctl_{tok}"
    leader = StripeLeader(ctl_name, 1, min_bytes=32 << 10)
    eng = Engine(spec, budget_bytes=budget, context_len=160, chunk_bytes=256 << 10, shared_weights=blob_name, striper=leader)
    print("[leader] engine ready", flush=True)
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=helper, args=(ctl_name, 1, blob_name, eng.weights.shared.nbytes))
    p.start()
    eng.attach_striper([40], 8)
    print("[leader] helpers attached", flush=True)
    t0 = time.time()
    got = eng.generate([prompt], gen_len=8)
    print(f"[leader] generated {got.tokens[0]} in {time.time()-t0:.2f}s err={leader.error_seq()} striped={leader.striped_pieces}", flush=True)
    eng.close(); leader.close()
    print("[leader] closed", flush=True)
    p.join(60)
    print("[leader] helper exit code", p.exitcode, flush=True)
