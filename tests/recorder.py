"""A CPU stand-in for ``KvDataPath``: records every device seam the plugin
drives (the eight KV transitions of SURVEY.md Appendix C and the batch
launches) so CPU tests can check the sequence without a GPU."""


class Recorder:
    def __init__(self, batch_seconds=None, swap_seconds=0.2):
        self.log = []
        self.measure = False
        self.batch_seconds = batch_seconds
        self.swap_s = swap_seconds

    def _rec(self, name, st, *extra):
        self.log.append((name, st.spec.id, st.kv_tokens) + extra)

    def drop(self, st):
        self._rec("drop", st)

    def swap_out_begin(self, st):
        self._rec("swap_out_begin", st)

    def swap_out_done(self, st):
        self._rec("swap_out_done", st)

    def swap_in_begin(self, st):
        self._rec("swap_in_begin", st)

    def swap_in_done(self, st):
        self._rec("swap_in_done", st)

    def release(self, st, where):
        self._rec("release", st, where.value)

    def launch_batch(self, members):
        self.log.append(("batch",) + tuple((m.state.spec.id, m.segment_index, m.prior_location.value,
                                            m.prior_kv_tokens) for m in members))
        if self.measure:
            return [self.batch_seconds * (1 + i % 3) for i, _ in enumerate(members)]
        return None

    def swap_seconds(self, state, direction):
        return self.swap_s

    def synchronize(self):
        pass

    def audit(self, states):
        pass

    def summary(self):
        return {"batches": sum(1 for e in self.log if e[0] == "batch")}
